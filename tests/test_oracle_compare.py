"""Pins of the oracle's encrypted comparison and scenario tail (NEXT-3, R29; not gpu).

(1) the paper's degree table kappa -> n and its PS split n = 13 -> (d1, d2) = (2, 4)
    (P:L727); the split is minimal by brute force over all (d1, d2);
(2) Chebyshev coefficients = numpy's chebinterpolate of f(x) = 1/2 (sign(x - delta) + 1)
    (library routine, first-kind points) and interpolate f at the n + 1 nodes (closed form);
(3) ChebyshevCompare decrypts to the plain series sum_i c_i T_i(x) (numpy chebval) on every
    slot, at the minimum multiplicative depth ceil(log2(n + 1)) (4 for n = 13), for the
    paper's degree (d1 = 2) and for n = 5 (d1 = 3: the odd baby power T3 = 2 T1 T2 - T1);
(3b) the fused Relinearize + Rescale (one rounding by P q_{ell-1}, the CUDA path's form): with
    d2 = 0 it is exactly the textbook Rescale of (d0, d1), and in general it equals Relinearize
    then Rescale bit for bit (mixed-radix identity) and decodes to the product of the slots;
(4) membership: every slot of RotateAndSum(sum of the inputs) decrypts to the sum of all
    decrypted input slots (a linear identity, independent of the evaluation);
(5) end to end on the flat scan (C1 database): compare(scan) decodes to chebval(cosine).
"""
import math

import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb

from synth_inputs import CONFIGS, make_dataset

D45 = 2.0 ** 45


def _f(delta):
    return lambda x: np.where(np.asarray(x) >= delta, 1.0, 0.0)


def test_degree_table_and_ps_split(oracle_mod):
    assert [oracle_mod.cheb_degree(k) for k in (7, 8, 9, 10)] == [5, 13, 27, 59]
    assert oracle_mod.cheb_degree(6) == 0
    assert oracle_mod.ps_split(13) == (2, 4)
    for n in (2, 3, 5, 13, 27, 59, 100):
        d1, d2 = oracle_mod.ps_split(n)
        assert d1 * 2 ** (d2 - 1) >= n
        best = min(a + b for a in range(1, n + 1) for b in range(1, 12) if a * 2 ** (b - 1) >= n)
        assert d1 + d2 == best


@pytest.mark.parametrize("delta,n", [(0.5, 13), (0.0, 13), (-0.3, 5), (0.8, 27)])
def test_coefficients(oracle_mod, delta, n):
    c = oracle_mod.cheb_coeffs(delta, n)
    ref = npcheb.chebinterpolate(_f(delta), n)
    assert np.abs(c - ref).max() < 1e-13
    xk = np.cos(np.pi * (np.arange(n + 1) + 0.5) / (n + 1))
    assert np.abs(npcheb.chebval(xk, c) - _f(delta)(xk)).max() < 1e-12


@pytest.fixture(scope="module")
def ring6(oracle_mod):
    o = oracle_mod.Oracle(10, 6, seed=5)
    s, s_ntt = o.secret_key()
    return o, s_ntt, o.relin_key(s_ntt)


def _encrypt_slots(o, s_ntt, z, ell, seed):
    return o.encrypt(s_ntt, o.encode(z, D45, ell), seed)


@pytest.mark.parametrize("n,delta", [(13, 0.5), (5, -0.2)])
def test_compare_evaluates_the_series(oracle_mod, ring6, n, delta):
    o, s_ntt, rlk = ring6
    rng = np.random.default_rng(n)
    z = rng.uniform(-1, 1, o.ns)
    z[:4] = [-1.0, 1.0, delta, 0.0]
    ell = 5                                   # the scan's output level at L = 6
    ct = _encrypt_slots(o, s_ntt, z, ell, 9)
    c = oracle_mod.cheb_coeffs(delta, n)
    out, scale = o.cheb_compare(ct, D45, c, rlk)
    assert out.shape[1] == 1                  # evaluated top-down to the last limb (R29)
    got = o.decode(o.decrypt(s_ntt, out), scale)
    want = npcheb.chebval(z, c)
    assert np.abs(got - want).max() < 1e-5
    # the approximation itself separates the far sides of the threshold
    far = np.abs(z - delta) > 0.4
    assert np.abs(got[far] - _f(delta)(z[far])).max() < 0.2


@pytest.mark.parametrize("n", [5, 13])
def test_compare_uses_the_minimum_depth(oracle_mod, ring6, n):
    """A degree-n polynomial needs ceil(log2(n + 1)) multiplicative levels (each product at
    most doubles the degree): the evaluation succeeds with exactly that many levels above q_0
    and reports OR_E_RANGE with one fewer."""
    o, s_ntt, rlk = ring6
    depth = math.ceil(math.log2(n + 1))
    c = oracle_mod.cheb_coeffs(0.3, n)
    z = np.random.default_rng(n).uniform(-1, 1, o.ns)
    ok = _encrypt_slots(o, s_ntt, z, depth + 1, 4)
    out, scale = o.cheb_compare(ok, D45, c, rlk)
    assert out.shape[1] == 1
    assert np.abs(o.decode(o.decrypt(s_ntt, out), scale) - npcheb.chebval(z, c)).max() < 1e-5
    short = _encrypt_slots(o, s_ntt, z, depth, 4)
    with pytest.raises(oracle_mod.OracleError) as e:
        o.cheb_compare(short, D45, c, rlk)
    assert e.value.code == oracle_mod.OR_E_RANGE


def test_fused_relin_rescale(oracle_mod, ring6):
    o, s_ntt, rlk = ring6
    rng = np.random.default_rng(21)
    ell = 4
    za, zb = rng.uniform(-1, 1, o.ns), rng.uniform(-1, 1, o.ns)
    a = _encrypt_slots(o, s_ntt, za, ell, 31)
    b = _encrypt_slots(o, s_ntt, zb, ell, 32)
    mods = [int(m) for m in o.p.moduli[:ell]]
    S3 = np.zeros((3, ell, o.n), dtype=np.uint64)
    for l, q in enumerate(mods):   # tensor in the NTT domain (pointwise), Python ints
        a0, a1 = a[0, l].astype(object), a[1, l].astype(object)
        b0, b1 = b[0, l].astype(object), b[1, l].astype(object)
        S3[0, l] = (a0 * b0 % q).astype(np.uint64)
        S3[1, l] = ((a0 * b1 + a1 * b0) % q).astype(np.uint64)
        S3[2, l] = (a1 * b1 % q).astype(np.uint64)
    # d2 = 0: exactly the textbook rescale of (d0, d1)
    Z = S3.copy()
    Z[2] = 0
    assert (o.relin_rescale(Z, rlk) == o.rescale(np.ascontiguousarray(S3[:2]))).all()
    # general: bit-identical to Relinearize then Rescale (mixed-radix identity of the two centred
    # lifts, R29), at every level, on the product and on uniform random residues
    assert (o.relin_rescale(S3, rlk) == o.rescale(o.relinearize(S3, rlk))).all()
    fused = o.relin_rescale(S3, rlk)
    scale = D45 * D45 / mods[ell - 1]
    assert np.abs(o.decode(o.decrypt(s_ntt, fused), scale) - za * zb).max() < 1e-6
    for e in (2, 3, 5):
        R = np.stack([np.stack([rng.integers(0, m, o.n, dtype=np.uint64) for m in o.p.moduli[:e]])
                      for _ in range(3)])
        assert (o.relin_rescale(R, rlk) == o.rescale(o.relinearize(R, rlk))).all(), e


def test_membership_sums_every_slot(oracle_mod, ring6):
    o, s_ntt, rlk = ring6
    rng = np.random.default_rng(3)
    zs = [rng.uniform(0, 1, o.ns) * 1e-3 for _ in range(3)]
    cts = np.stack([_encrypt_slots(o, s_ntt, z, 2, 40 + i) for i, z in enumerate(zs)])
    steps = [1 << k for k in range(o.log_n - 1)]
    st, keys = o.keyset(s_ntt, steps)
    out = o.membership(cts, st, keys)
    got = o.decode(o.decrypt(s_ntt, out), D45)
    dec = sum(o.decode(o.decrypt(s_ntt, cts[i]), D45) for i in range(3))
    assert np.abs(got - dec.sum()).max() < 1e-6
    with pytest.raises(oracle_mod.OracleError):
        o.membership(cts, st[:-1], keys[:-1])


def test_identification_end_to_end(oracle_mod):
    """Flat scan at L = 6, then ChebyshevCompare: decodes to chebval(cosine) per vector."""
    cfg = CONFIGS["C1"]
    o = oracle_mod.Oracle(cfg.log_n, 6, seed=1)
    s, s_ntt = o.secret_key()
    rlk = o.relin_key(s_ntt)
    db, q, pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    st, keys = o.keyset(s_ntt, o.rotation_steps_flat(cfg.dim, cfg.n1))
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), D45, o.L), 1000)
    r = o.baby_steps(qct, cfg.n1, st, keys)
    D = o.enroll_aggregate_flat(o.normalize_rows(db), 0, cfg.num_vectors, cfg.n1, 0)
    out = o.scan_aggregate_flat(r, cfg.n1, cfg.dim, D, st, keys)
    delta = 0.5
    c = oracle_mod.cheb_coeffs(delta, 13)
    cmp_ct, scale = o.cheb_compare(out, D45, c, rlk)
    assert cmp_ct.shape[1] == 1
    z = o.decode(o.decrypt(s_ntt, cmp_ct), scale)
    d = db.astype(np.float64)
    cos = d @ q.astype(np.float64) / (np.linalg.norm(d, axis=1) * np.linalg.norm(q.astype(np.float64)))
    got = z[: cfg.num_vectors]          # flat packing, one aggregate: slot v = vector v (R27)
    assert np.abs(got - npcheb.chebval(cos, c)).max() < 1e-5
    assert (got[pos] > 0.8).all() and np.delete(got, pos).max() < 0.3


@pytest.mark.parametrize("n", [1, 2, 3])
def test_compare_low_degrees(oracle_mod, ring6, n):
    """Degenerate Paterson-Stockmeyer shapes: n = 1 (d1 = 1: a single scalar product),
    n = 2 (d1 = 2, one giant power), n = 3; each decodes to the series."""
    o, s_ntt, rlk = ring6
    z = np.random.default_rng(40 + n).uniform(-1, 1, o.ns)
    c = np.array([0.25, -0.5, 0.75, 0.125][: n + 1])
    out, scale = o.cheb_compare(_encrypt_slots(o, s_ntt, z, 4, 5), D45, c, rlk)
    assert out.shape[1] == 1
    assert np.abs(o.decode(o.decrypt(s_ntt, out), scale) - npcheb.chebval(z, c)).max() < 1e-5


def test_compare_constant_series_is_rejected(oracle_mod, ring6):
    """delta <= -1: f = 1 on the whole interval, the interpolant is the constant 1 and there is
    nothing encrypted to evaluate (the CUDA path returns HD_E_INVALID_ARG alike)."""
    o, s_ntt, rlk = ring6
    c = oracle_mod.cheb_coeffs(-1.5, 13)
    assert abs(c[0] - 1.0) < 1e-15 and np.abs(c[1:]).max() < 1e-15
    with pytest.raises(oracle_mod.OracleError) as e:
        o.cheb_compare(_encrypt_slots(o, s_ntt, np.zeros(o.ns), 5, 6), D45, np.array([1.0] + [0.0] * 13), rlk)
    assert e.value.code == oracle_mod.OR_E_ARG


def test_online_aggregation_is_the_sum_of_the_scans(oracle_mod):
    """Alg. online-aggr: the scan of the aggregated diagonals decrypts to the sum
    of the per-aggregate scans (the scan is linear), slot by slot, within the CKKS noise."""
    from synth_inputs import Config
    cfg = Config("agg", 12, 64, 2500, 8, index=11)   # 3 aggregates of 1024 vectors, the last ragged
    o = oracle_mod.Oracle(cfg.log_n, cfg.limbs, seed=1)
    s, s_ntt = o.secret_key()
    db, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    st, keys = o.keyset(s_ntt, o.rotation_steps(cfg.dim, cfg.n1))
    r = o.baby_steps(o.encrypt(s_ntt, o.encode(o.query_slots(q), D45, o.L), 1000), cfg.n1, st, keys)
    U = o.normalize_rows(db)
    per = (o.ns // cfg.dim // 2) * cfg.dim
    # Alg. enroller_bsgs builds aggregates in (ctA, ctB) pairs from one temporary: pass the pair's rows
    Ds = [o.enroll_aggregate(U[(a - a % 2) * per:(a - a % 2 + 2) * per], (a - a % 2) * per, cfg.num_vectors,
                             cfg.n1, a) for a in range(3)]
    Dsum = o.aggregate_diagonals(Ds)
    mods = np.array(o.p.moduli[:o.L], dtype=object)[:, None]
    assert ((sum(D.astype(object) for D in Ds) % mods) == Dsum.astype(object)).all()   # residue-wise sum
    z_sum = o.decode(o.decrypt(s_ntt, o.scan_aggregate(r, cfg.n1, cfg.dim, Dsum, st, keys)), D45)
    z_parts = sum(o.decode(o.decrypt(s_ntt, o.scan_aggregate(r, cfg.n1, cfg.dim, D, st, keys)), D45) for D in Ds)
    assert np.abs(z_sum - z_parts).max() < 1e-6


def test_compare_to_two_limbs(oracle_mod, ring6):
    """The result requested at 2 limbs (membership headroom, R29): same series, one level more left."""
    o, s_ntt, rlk = ring6
    z = np.random.default_rng(77).uniform(-1, 1, o.ns)
    c = oracle_mod.cheb_coeffs(0.5, 13)
    out, scale = o.cheb_compare(_encrypt_slots(o, s_ntt, z, 6, 8), D45, c, rlk, out_limbs=2)
    assert out.shape[1] == 2
    assert np.abs(o.decode(o.decrypt(s_ntt, out), scale) - npcheb.chebval(z, c)).max() < 1e-5
    with pytest.raises(oracle_mod.OracleError):   # 5 limbs leave no room for degree 13 at 2 limbs
        o.cheb_compare(_encrypt_slots(o, s_ntt, z, 5, 8), D45, c, rlk, out_limbs=2)
