"""Pins of the oracle's encrypted-database mode (NEXT-1, R26; not gpu).

(1) public-key encryption: decrypt(Enc_pk(m)) - m = v e + e0 + e1 s, a small centred
    polynomial (|.| <= 21 (||v||_1 + 1 + ||s||_1)); the sum of two encryptions decrypts
    to the sum of the messages;
(2) the degree-2 giant-step sum is the exact tensor product: d0 + d1 s + d2 s^2 =
    sum_i dec(r_i) dec(Dct_k) in the ring (pointwise in the NTT domain), bit for bit;
(3) relinearisation: dec(Relin(d0, d1, d2)) - (d0 + d1 s + d2 s^2) is the key-switching
    noise (< 2^20 at the plaintext level of the toy ring);
(4) encrypted scan end to end: scores = brute-force cosine within 1e-6, planted matches on
    top, and the same scores as the plaintext-diagonal scan (<= 1e-6).
"""
import numpy as np
import pytest

from synth_inputs import CONFIGS, make_dataset
from tests.test_oracle_scan import _centred_coeffs, _cos

D45 = 2.0 ** 45


def _dec_poly(o, s_ntt, ct):
    """Ring decryption in NTT form, any degree: sum_d c_d s^d per limb (pointwise)."""
    mods = o.p.moduli
    deg = ct.shape[0]
    out = np.zeros(ct.shape[1:], dtype=object)
    for l in range(ct.shape[1]):
        q = mods[l]
        s = [int(x) for x in s_ntt[l]]
        for t in range(o.n):
            acc, sp = 0, 1
            for d in range(deg):
                acc += int(ct[d, l, t]) * sp
                sp = sp * s[t] % q
            out[l, t] = acc % q
    return out


@pytest.fixture(scope="module")
def toy(oracle_mod):
    o = oracle_mod.Oracle(9, 3, seed=21)
    s, s_ntt = o.secret_key()
    return o, s, s_ntt, o.public_key(s_ntt)


def test_public_key_encryption_noise(toy):
    o, s, s_ntt, pk = toy
    z = np.random.default_rng(1).uniform(-1, 1, o.ns)
    m = o.encode(z, D45, o.L)
    ct = o.encrypt_pk(pk, m, 77, 5)
    err = _centred_coeffs(o, (o.decrypt(s_ntt, ct).astype(object) - m.astype(object)) % np.array(
        o.p.moduli[:o.L], dtype=object)[:, None])
    bound = 21 * (o.n + 1 + int(np.abs(s).sum()))   # ||v||_1 <= n
    assert 0 < max(abs(e) for e in err) <= bound
    m2 = o.encode(z[::-1].copy(), D45, o.L)
    ct2 = o.encrypt_pk(pk, m2, 77, 6)
    summ = (ct.astype(object) + ct2.astype(object)) % np.array(o.p.moduli[:o.L], dtype=object)[None, :, None]
    got = o.decode(o.decrypt(s_ntt, summ.astype(np.uint64)), D45)
    assert np.abs(got - (z + z[::-1])).max() < 1e-6
    # distinct object ids draw distinct randomness
    assert not (o.encrypt_pk(pk, m, 77, 5) == o.encrypt_pk(pk, m, 77, 6)).all()


def test_degree2_giant_sum_is_the_tensor_product(toy):
    o, s, s_ntt, pk = toy
    rng = np.random.default_rng(3)
    n1, N, L = 4, 16, o.L
    mods = np.array(o.p.moduli[:L], dtype=np.uint64)[None, None, :, None]
    r = (rng.integers(0, 2 ** 62, size=(n1, 2, L, o.n), dtype=np.uint64) % mods).astype(np.uint64)
    D = (rng.integers(0, 2 ** 62, size=(N, 2, L, o.n), dtype=np.uint64) % mods).astype(np.uint64)
    for j in (-2, 0, 1):
        S3 = o.giant_sum_ct(r, n1, N, D, j)
        lhs = _dec_poly(o, s_ntt, S3)
        rhs = np.zeros_like(lhs)
        i_lo, i_hi = max(0, -j * n1 - N // 2), min(n1 - 1, N // 2 - 1 - j * n1)
        for i in range(i_lo, i_hi + 1):
            k = ((j * n1 + i) % N + N) % N
            rhs = rhs + _dec_poly(o, s_ntt, r[i]) * _dec_poly(o, s_ntt, D[k])
        rhs = rhs % np.array(o.p.moduli[:L], dtype=object)[:, None]
        assert (lhs == rhs).all(), j


def test_relinearisation_noise(toy):
    o, s, s_ntt, pk = toy
    rlk = o.relin_key(s_ntt)
    z1 = np.random.default_rng(4).uniform(-1, 1, o.ns)
    z2 = np.random.default_rng(5).uniform(-1, 1, o.ns)
    c1 = o.encrypt_pk(pk, o.encode(z1, D45, o.L), 9, 1)
    c2 = o.encrypt_pk(pk, o.encode(z2, D45, o.L), 9, 2)
    mods = np.array(o.p.moduli[:o.L], dtype=object)[:, None]
    a0, a1, b0, b1 = (x.astype(object) for x in (c1[0], c1[1], c2[0], c2[1]))
    S3 = np.stack([(a0 * b0) % mods, (a0 * b1 + a1 * b0) % mods, (a1 * b1) % mods]).astype(np.uint64)
    out = o.relinearize(S3, rlk)
    want = _dec_poly(o, s_ntt, S3)
    got = o.decrypt(s_ntt, out).astype(object)
    diff = _centred_coeffs(o, ((got - want) % mods).astype(np.uint64))
    assert max(abs(d) for d in diff) < 2 ** 20
    # and the product decodes to z1 z2 at scale D45^2
    dec = o.decode(o.decrypt(s_ntt, o.rescale(out)), D45 * D45 / o.p.moduli[o.L - 1])
    assert np.abs(dec - z1 * z2).max() < 1e-6


def test_encrypted_scan_scores(oracle_mod):
    cfg = CONFIGS["C1"]
    o = oracle_mod.Oracle(cfg.log_n, cfg.limbs, seed=1)
    db, q, pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    s, s_ntt = o.secret_key()
    pk, rlk = o.public_key(s_ntt), o.relin_key(s_ntt)
    steps, keys = o.keyset(s_ntt, o.rotation_steps(cfg.dim, cfg.n1))
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), D45, o.L), 1000)
    r = o.baby_steps(qct, cfg.n1, steps, keys)
    U = o.normalize_rows(db)
    Dct = o.enroll_aggregate_encrypted(U, 0, cfg.num_vectors, cfg.n1, 0, pk, 4242)
    Dpt = o.enroll_aggregate(U, 0, cfg.num_vectors, cfg.n1, 0)
    for k in (0, cfg.dim - 1):   # each encrypted diagonal decrypts to its plaintext (+ noise)
        diff = _centred_coeffs(o, ((o.decrypt(s_ntt, Dct[k]).astype(object) - Dpt[k].astype(object))
                                   % np.array(o.p.moduli[:o.L], dtype=object)[:, None]).astype(np.uint64))
        assert max(abs(d) for d in diff) < 2 ** 20
    out = o.scan_aggregate_ct(r, cfg.n1, cfg.dim, Dct, steps, keys, rlk)
    sc = o.decrypt_scores(s_ntt, out, cfg.dim, 0, cfg.num_vectors)[:cfg.num_vectors]
    assert np.abs(sc - _cos(db, q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:len(pos)]) == sorted(pos.tolist())
    sc_pt = o.decrypt_scores(s_ntt, o.scan_aggregate(r, cfg.n1, cfg.dim, Dpt, steps, keys), cfg.dim, 0,
                             cfg.num_vectors)[:cfg.num_vectors]
    assert np.abs(sc - sc_pt).max() < 1e-6
