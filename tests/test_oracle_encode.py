"""Pins for the CKKS encoder / encryption / key switching of the oracle (not gpu).

Encoding is checked against the O(n^2) canonical embedding (the
slot j of m is m(zeta^{5^j}) / Delta with zeta = exp(2 pi i / 2n)), rotations
against the in-the-clear slot permutation, rescale/ModDown
against exact integer identities and an analytic noise bound.
"""
import numpy as np
import pytest

D45 = 2.0 ** 45


def _embed(coef, n, delta):
    """Canonical embedding at zeta^{5^j}, j < n/2 -- plain definition."""
    ns = n // 2
    zeta_pows = [pow(5, j, 2 * n) for j in range(ns)]
    k = np.arange(n)
    out = np.empty(ns, dtype=np.complex128)
    c = coef.astype(np.float64)
    for j, e in enumerate(zeta_pows):
        out[j] = np.sum(c * np.exp(2j * np.pi * ((e * k) % (2 * n)) / (2 * n)))
    return out / delta


@pytest.mark.parametrize("log_n", [4, 8, 10])
def test_encode_is_inverse_canonical_embedding(oracle_mod, log_n):
    o = oracle_mod.Oracle(log_n, 3)
    rng = np.random.default_rng(log_n)
    z = rng.uniform(-1, 1, o.ns)
    coef = o.encode_coeffs(z, D45)
    emb = _embed(coef, o.n, D45)
    # rounding error of each coefficient is <= 1/2 -> slot error <= n/2/Delta
    assert np.abs(emb.real - z).max() < o.n / D45
    assert np.abs(emb.imag).max() < o.n / D45   # real slots -> conjugate-symmetric embedding
    # residues are the coefficients mod q_l, NTT'd
    pt = o.encode(z, D45, 3)
    for l, m in enumerate(o.p.moduli[:3]):
        ref = np.array([int(c) % m for c in coef.tolist()], dtype=np.uint64)
        assert (o.ntt(pt[l], l, inverse=True) == ref).all()


def test_encode_decode_roundtrip(oracle_mod):
    o = oracle_mod.Oracle(12, 3)
    z = np.random.default_rng(5).uniform(-1, 1, o.ns)
    for nl in (1, 2, 3):
        assert np.abs(o.decode(o.encode(z, D45, nl), D45) - z).max() < 1e-9


@pytest.fixture(scope="module")
def toy(oracle_mod):
    o = oracle_mod.Oracle(12, 3, seed=1)
    s, s_ntt = o.secret_key()
    return o, s, s_ntt


def test_encrypt_decrypt(toy):
    o, s, s_ntt = toy
    z = np.random.default_rng(6).uniform(-1, 1, o.ns)
    pt = o.encode(z, D45, 3)
    ct = o.encrypt(s_ntt, pt, 1000)
    dec = o.decrypt(s_ntt, ct)
    # decrypt - pt = e (fresh CBD(21) noise, |e_j| <= 21)
    for l, m in enumerate(o.p.moduli[:3]):
        e = o.ntt((dec[l].astype(object) - pt[l].astype(object)) % m, l, inverse=True).astype(object)
        e = [(int(x) if int(x) <= m // 2 else int(x) - m) for x in e]
        assert max(abs(x) for x in e) <= 21
        assert np.std(e) > 2.5   # CBD(21): sigma = sqrt(10.5) ~ 3.24
    assert np.abs(o.decode(dec, D45) - z).max() < 1e-9


@pytest.mark.parametrize("step", [1, 5, 64, 1984])
def test_rotation_is_slot_shift(toy, step):
    o, s, s_ntt = toy
    z = np.random.default_rng(step).uniform(-1, 1, o.ns)
    ct = o.encrypt(s_ntt, o.encode(z, D45, 3), 1001)
    key = o.rotation_key(s_ntt, step)
    for ell in (3, 2):
        c = ct if ell == 3 else np.ascontiguousarray(ct[:, :2])
        rot = o.rotate(c, key, step)
        dec = o.decode(o.decrypt(s_ntt, rot), D45)
        assert np.abs(dec - np.roll(z, -step)).max() < 1e-7   # Rot_r(x)[t] = x[t + r]  (R7)
        # key-switch noise bound on the integer plaintext: |error coeff| < 2^20
        ref = o.decrypt(s_ntt, c)
        g = o.galois_elt(step)
        for l in range(ell):
            m = o.p.moduli[l]
            want = o.automorph_ntt(g, ref[l])
            got = o.decrypt(s_ntt, rot)[l]
            diff = o.ntt((got.astype(object) - want.astype(object)) % m, l, inverse=True)
            diff = np.array([(int(x) if int(x) <= m // 2 else int(x) - m) for x in diff])
            assert np.abs(diff).max() < 2 ** 20


def test_hoisted_equals_single_rotation(toy):
    o, s, s_ntt = toy
    z = np.random.default_rng(9).uniform(-1, 1, o.ns)
    ct = o.encrypt(s_ntt, o.encode(z, D45, 3), 1002)
    key = o.rotation_key(s_ntt, 3)
    dig = o.modup(np.ascontiguousarray(ct[1]))
    assert (o.rotate_hoisted(ct, dig, key, 3) == o.rotate(ct, key, 3)).all()


def test_rescale_exact_rounding(toy):
    """X = q_last * x + e with |e| < q_last/2 -> Rescale(X) = x exactly (R12)."""
    o, s, s_ntt = toy
    n = o.n
    rng = np.random.default_rng(10)
    q = o.p.moduli
    ql = q[2]
    x = rng.integers(-2**40, 2**40, size=(2, n)).astype(object)
    e = rng.integers(-(ql // 2) + 1, ql // 2, size=(2, n)).astype(object)
    X = x * ql + e
    ct = np.zeros((2, 3, n), dtype=np.uint64)
    for p_ in range(2):
        for l in range(3):
            ct[p_, l] = o.ntt(np.array([int(v) % q[l] for v in X[p_]], dtype=np.uint64), l)
    out = o.rescale(ct)
    for p_ in range(2):
        for l in range(2):
            got = o.ntt(out[p_, l], l, inverse=True)
            assert [int(v) for v in got] == [int(v) % q[l] for v in x[p_]]
