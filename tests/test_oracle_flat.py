"""Pins of the oracle's flat pre-rotated layout (NEXT-2, R27: BSGS-RTX-TBE; not gpu).

(1) an independent numpy plaintext-slot shadow of the flat schedule -- HyDia packing
    (Eq. equ:diag), enroller pre-rotation diag'_k = Rot_{-j n1}(diag_k)
    (Eq. eq:prerotation), S_j = sum_i Rot_i(q) (.) diag'_{j n1 + i},
    y = sum_j Rot_{j n1}(S_j) -- equals brute-force cosine;
(2) the oracle's slot vectors equal the shadow's, and Rot_{j n1}(diag'_k) = diag_k;
(3) the key set is the paper's S_baby u S_giant ((n1-1) + (n2-1) keys);
(4) encrypted flat scan: scores = cosine within 1e-6, planted matches on top, and the
    same scores as the replicated-layout scan.
"""
import numpy as np
import pytest

from synth_inputs import CONFIGS, make_dataset
from tests.test_oracle_scan import _cos

D45 = 2.0 ** 45


def rot(x, r):
    """Rot_r(x)[t] = x[t + r] (R7)."""
    return np.roll(x, -r)


def shadow_flat_diag(U, N, ns, agg, k, n1, prerotate=True):
    M = ns // N
    d = np.zeros(ns)
    for b in range(M):
        for t in range(N):
            v = (agg * M + b) * N + t
            if v < U.shape[0]:
                d[b * N + t] = U[v, (t + k) % N]
    return rot(d, -(k // n1) * n1) if prerotate else d


def shadow_flat_scan(U, u, N, ns, n1, agg):
    qrep = np.tile(u, ns // N)
    y = np.zeros(ns)
    for j in range(-(-N // n1)):
        S = np.zeros(ns)
        for i in range(n1):
            if j * n1 + i < N:
                S += rot(qrep, i) * shadow_flat_diag(U, N, ns, agg, j * n1 + i, n1)
        y += rot(S, j * n1)
    return y


@pytest.mark.parametrize("ns,N,K,n1", [(1024, 64, 200, 8), (1024, 64, 64, 16), (256, 16, 40, 4),
                                        (512, 32, 100, 32), (512, 32, 100, 1), (256, 16, 50, 3)])
def test_flat_shadow_equals_cosine(ns, N, K, n1):
    rng = np.random.default_rng(K * n1)
    db = rng.integers(-99, 100, size=(K, N)).astype(np.float32)
    q = rng.integers(-99, 100, size=N).astype(np.float32)
    U = db.astype(np.float64) / np.linalg.norm(db.astype(np.float64), axis=1, keepdims=True)
    u = q.astype(np.float64) / np.linalg.norm(q.astype(np.float64))
    M = ns // N
    A = -(-K // (M * N))
    got = []
    for a in range(A):
        y = shadow_flat_scan(U, u, N, ns, n1, a)
        got.append(y[:min(M * N, K - a * M * N)])
    assert np.abs(np.concatenate(got) - _cos(db, q)).max() < 1e-12


def test_oracle_flat_slots_equal_shadow_and_prerotation_identity(oracle_mod):
    o = oracle_mod.Oracle(9, 3)   # ns = 256
    rng = np.random.default_rng(5)
    K, N, n1 = 40, 16, 4          # M = 16 groups per ct; 3 groups -> one partial aggregate
    U = o.normalize_rows(rng.integers(-99, 100, size=(K, N)).astype(np.float32))
    for k in range(N):
        z = o.enroll_slots_flat(U, 0, K, n1, 0, k)
        assert (z == shadow_flat_diag(U, N, o.ns, 0, k, n1)).all(), k
        assert (rot(z, (k // n1) * n1) == shadow_flat_diag(U, N, o.ns, 0, k, n1, prerotate=False)).all(), k


@pytest.mark.parametrize("N,n1", [(512, 128), (512, 23), (64, 8), (16, 16)])
def test_flat_key_census(oracle_mod, N, n1):
    o = oracle_mod.Oracle(12, 3)
    steps = o.rotation_steps_flat(N, n1)
    n2 = -(-N // n1)
    assert len(steps) == (n1 - 1) + (n2 - 1)
    assert set(steps) == set(range(1, n1)) | {j * n1 for j in range(1, n2)}
    if (N, n1) == (512, 23):
        assert len(steps) == 44  # the paper's count at n1 = n2 = 23


def test_flat_encrypted_scan_scores(oracle_mod):
    cfg = CONFIGS["C1"]
    o = oracle_mod.Oracle(cfg.log_n, cfg.limbs, seed=1)
    db, q, pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    s, s_ntt = o.secret_key()
    steps, keys = o.keyset(s_ntt, o.rotation_steps_flat(cfg.dim, cfg.n1))
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), D45, o.L), 1000)
    r = o.baby_steps(qct, cfg.n1, steps, keys)
    U = o.normalize_rows(db)
    D = o.enroll_aggregate_flat(U, 0, cfg.num_vectors, cfg.n1, 0)
    out = o.scan_aggregate_flat(r, cfg.n1, cfg.dim, D, steps, keys)
    sc = o.decrypt_scores_flat(s_ntt, out, cfg.dim, 0, cfg.num_vectors)[:cfg.num_vectors]
    assert np.abs(sc - _cos(db, q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:len(pos)]) == sorted(pos.tolist())


def test_flat_encrypted_database_scan(oracle_mod):
    """BSGS-RTX-TBE with encrypted diagonals (the paper's GPU setting, P:L883-905 with
    P:L119): the degree-2 flat giant sum is the exact tensor product of the decrypted
    operands, and the scan decodes to cosine within 1e-6 with the planted matches on top."""
    from tests.test_oracle_encdb import _dec_poly
    cfg = CONFIGS["C1"]
    o = oracle_mod.Oracle(cfg.log_n, cfg.limbs, seed=1)
    db, q, pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    s, s_ntt = o.secret_key()
    pk, rlk = o.public_key(s_ntt), o.relin_key(s_ntt)
    steps, keys = o.keyset(s_ntt, o.rotation_steps_flat(cfg.dim, cfg.n1))
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), D45, o.L), 1000)
    r = o.baby_steps(qct, cfg.n1, steps, keys)
    Dct = o.enroll_aggregate_flat_encrypted(o.normalize_rows(db), 0, cfg.num_vectors, cfg.n1, 0, pk, 77)
    j = 1
    S3 = o.giant_sum_ct_flat(r, cfg.n1, cfg.dim, Dct, j)
    rhs = sum(_dec_poly(o, s_ntt, r[i]) * _dec_poly(o, s_ntt, Dct[j * cfg.n1 + i]) for i in range(cfg.n1))
    rhs = rhs % np.array(o.p.moduli[:o.L], dtype=object)[:, None]
    assert (_dec_poly(o, s_ntt, S3) == rhs).all()
    out = o.scan_aggregate_flat_ct(r, cfg.n1, cfg.dim, Dct, steps, keys, rlk)
    sc = o.decrypt_scores_flat(s_ntt, out, cfg.dim, 0, cfg.num_vectors)[:cfg.num_vectors]
    assert np.abs(sc - _cos(db, q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:len(pos)]) == sorted(pos.tolist())


def test_flat_tbs_server_prerotation(oracle_mod):
    """BSGS-RTX-TBS: plain flat diagonals encrypted by the enroller, pre-rotated
    homomorphically by the server with the negative giant-step keys.  Each pre-rotated
    ciphertext decrypts to the enroller-side pre-rotated (TBE) plaintext within the
    key-switching noise, and the scan decodes to cosine like TBE."""
    from tests.test_oracle_scan import _centred_coeffs
    cfg = CONFIGS["C1"]
    o = oracle_mod.Oracle(cfg.log_n, cfg.limbs, seed=1)
    db, q, pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    N, n1 = cfg.dim, cfg.n1
    s, s_ntt = o.secret_key()
    pk, rlk = o.public_key(s_ntt), o.relin_key(s_ntt)
    neg = [o.ns - j * n1 for j in range(1, -(-N // n1))]
    steps, keys = o.keyset(s_ntt, sorted(set(o.rotation_steps_flat(N, n1)) | set(neg)))
    U = o.normalize_rows(db)
    Dtbs = o.prerotate_tbs(o.enroll_aggregate_flat_tbs(U, 0, cfg.num_vectors, n1, 0, pk, 5), n1, steps, keys)
    Dtbe = o.enroll_aggregate_flat(U, 0, cfg.num_vectors, n1, 0)   # plaintext pre-rotated by the enroller
    mods = np.array(o.p.moduli[:o.L], dtype=object)[:, None]
    for k in (0, n1, N - 1):
        diff = _centred_coeffs(o, ((o.decrypt(s_ntt, Dtbs[k]).astype(object) - Dtbe[k].astype(object)) % mods)
                               .astype(np.uint64))
        assert max(abs(d) for d in diff) < 2 ** 20, k
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), D45, o.L), 1000)
    r = o.baby_steps(qct, n1, steps, keys)
    out = o.scan_aggregate_flat_ct(r, n1, N, Dtbs, steps, keys, rlk)
    sc = o.decrypt_scores_flat(s_ntt, out, N, 0, cfg.num_vectors)[:cfg.num_vectors]
    assert np.abs(sc - _cos(db, q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:len(pos)]) == sorted(pos.tolist())
