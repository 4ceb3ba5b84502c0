"""GPU parity of the encrypted comparison and the scenario tails (NEXT-3, R29): the CUDA path
through the C ABI vs the CPU oracle, bit-exact on every residue (scan outputs at six limbs,
ChebyshevCompare of a batch of aggregates incl. a ragged tail, membership), equal scales, and
decrypted comparisons vs the plain Chebyshev series of the brute-force cosine."""
import dataclasses

import numpy as np
import pytest
from numpy.polynomial import chebyshev as npcheb

from synth_inputs import CONFIGS, ENC_SEED_BASE, make_dataset

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_00546_b200 as hd  # noqa: E402

D45 = 2.0 ** 45


def _cos(db, q):
    d = db.astype(np.float64)
    qq = q.astype(np.float64)
    return d @ qq / (np.linalg.norm(d, axis=1) * np.linalg.norm(qq))


class CmpRun:
    """C1 ring (2^12) at L = 6 limbs, flat packing, 5000 vectors -> 3 aggregates (last ragged)."""

    def __init__(self):
        cfg = dataclasses.replace(CONFIGS["C1"], limbs=6, num_vectors=5000)
        self.cfg = cfg
        self.ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
        self.o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
        self.db_vecs, self.q, self.pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
        scan_steps = [int(s) for s in self.ctx.rotation_steps(cfg.dim, cfg.n1, packing="flat")]
        self.mem_steps = [int(s) for s in self.ctx.membership_steps()]
        self.steps = sorted(set(scan_steps) | set(self.mem_steps))
        self.sk, self.evk = self.ctx.keygen(np.array(self.steps, np.int32))
        self.ctx.relin_keygen(self.sk, self.evk)
        self.qct = self.ctx.encrypt_query(self.sk, self.q, ENC_SEED_BASE)
        self.db = self.ctx.enroll(self.db_vecs, cfg.n1, packing="flat")
        self.outs = self.ctx.query(self.evk, self.db, self.qct)
        torch.cuda.synchronize()
        _, self.s_ntt = self.o.secret_key()
        self.ok_steps, self.ok_keys = self.o.keyset(self.s_ntt, self.steps)
        self.rlk = self.o.relin_key(self.s_ntt)
        z = self.o.query_slots(self.q)
        qct = self.o.encrypt(self.s_ntt, self.o.encode(z, D45, cfg.limbs), ENC_SEED_BASE)
        r = self.o.baby_steps(qct, cfg.n1, self.ok_steps, self.ok_keys)
        self.ref_outs = []
        per = self.o.ns
        for agg in range(len(self.outs)):
            v0, v1 = agg * per, min(cfg.num_vectors, (agg + 1) * per)
            D = self.o.enroll_aggregate_flat(self.o.normalize_rows(self.db_vecs[v0:v1]), v0, cfg.num_vectors,
                                             cfg.n1, agg)
            self.ref_outs.append(self.o.scan_aggregate_flat(r, cfg.n1, cfg.dim, D, self.ok_steps, self.ok_keys))
        self.cos = _cos(self.db_vecs, self.q)


@pytest.fixture(scope="module")
def run():
    return CmpRun()


def test_scan_bit_exact_at_six_limbs(run):
    assert len(run.outs) == 3
    for got, ref in zip(run.outs, run.ref_outs):
        assert got.limbs == 5 and (run.ctx.ciphertext_residues(got) == ref).all()
        assert run.ctx.ciphertext_scale(got) == D45


@pytest.mark.parametrize("delta,kappa", [(0.5, 8), (-0.2, 7)])
def test_compare_bit_exact(run, delta, kappa):
    n = hd.chebyshev_degree(kappa)
    c = hd.chebyshev_coefficients(delta, n)
    assert (c == oracle.cheb_coeffs(delta, n)).all()
    cmp = run.ctx.compare(run.evk, run.outs, c)
    torch.cuda.synchronize()
    for agg, (got, ref) in enumerate(zip(cmp, run.ref_outs)):
        want, scale = run.o.cheb_compare(ref, D45, c, run.rlk)
        assert got.limbs == want.shape[1] == 1   # evaluated top-down to q_0 (R29)
        assert (run.ctx.ciphertext_residues(got) == want).all(), agg
        assert run.ctx.ciphertext_scale(got) == scale


def test_identification_decodes_to_the_series(run):
    c = hd.chebyshev_coefficients(0.5, 13)
    cmp = run.ctx.compare(run.evk, run.outs, c)
    per = run.ctx.ns
    got = np.concatenate([run.ctx.decrypt_slots(run.sk, ct) for ct in cmp])[: run.cfg.num_vectors]
    assert np.abs(got - npcheb.chebval(run.cos, c)).max() < 1e-5
    far = np.abs(run.cos - 0.5) > 0.4      # the degree-13 series separates values far from delta
    assert (got[run.pos] > 0.8).all() and np.abs(got[far] - (run.cos[far] >= 0.5)).max() < 0.2
    assert per * len(cmp) >= run.cfg.num_vectors
    # in-place reuse of the outputs gives the same bits
    again = run.ctx.compare(run.evk, run.outs, c, outs=cmp)
    assert again[0] is cmp[0]
    ref = run.o.cheb_compare(run.ref_outs[1], D45, c, run.rlk)[0]
    assert (run.ctx.ciphertext_residues(again[1]) == ref).all()


def test_membership_bit_exact(run):
    c = hd.chebyshev_coefficients(0.5, 13)
    cmp = run.ctx.compare(run.evk, run.outs, c)
    mem = run.ctx.membership(run.evk, cmp)
    torch.cuda.synchronize()
    refs = np.stack([run.o.cheb_compare(r, D45, c, run.rlk)[0] for r in run.ref_outs])
    want = run.o.membership(refs, np.array(run.mem_steps, np.int32),
                            run.ok_keys[[run.steps.index(s) for s in run.mem_steps]])
    assert (run.ctx.ciphertext_residues(mem) == want).all()
    z = run.ctx.decrypt_slots(run.sk, mem)
    total = npcheb.chebval(run.cos, c).sum() + (len(cmp) * run.ctx.ns - run.cfg.num_vectors) * npcheb.chebval(0.0, c)
    assert np.abs(z - total).max() < 1e-3 * max(1.0, abs(total))


def test_compare_errors(run):
    c = hd.chebyshev_coefficients(0.5, 27)   # depth 5 > the 4 levels left
    with pytest.raises(hd.HDError) as e:
        run.ctx.compare(run.evk, run.outs, c)
    assert e.value.code == -6  # HD_E_LEVEL
    sk2, evk2 = run.ctx.keygen(np.array([1], np.int32))   # no relinearisation key
    with pytest.raises(hd.HDError) as e:
        run.ctx.compare(evk2, run.outs[:1], hd.chebyshev_coefficients(0.5, 13))
    assert e.value.code == -5  # HD_E_MISSING_KEY
    with pytest.raises(hd.HDError) as e:
        run.ctx.membership(evk2, run.outs[:1])
    assert e.value.code == -5


@pytest.mark.slow
def test_compare_at_bench_ring_size():
    """ChebyshevCompare at the bench's ring (2^16) and limb count (6), as a batch of 32
    ciphertexts (the bench's batch): bit-exact vs the oracle on an encrypted slot vector."""
    cfg = dataclasses.replace(CONFIGS["C4"], limbs=6)
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
    sk, evk = ctx.keygen(np.array([1], np.int32))
    ctx.relin_keygen(sk, evk)
    v = np.random.default_rng(11).integers(-99, 100, cfg.dim).astype(np.float32)
    cts = [ctx.encrypt_query(sk, v, ENC_SEED_BASE + 7)] * 32
    c = hd.chebyshev_coefficients(0.05, 13)
    out = ctx.compare(evk, cts, c)
    torch.cuda.synchronize()
    _, s_ntt = o.secret_key()
    oct_ = o.encrypt(s_ntt, o.encode(o.query_slots(v), D45, cfg.limbs), ENC_SEED_BASE + 7)
    assert (ctx.ciphertext_residues(cts[0]) == oct_).all()
    want, scale = o.cheb_compare(oct_, D45, c, o.relin_key(s_ntt))
    for k in (0, 31):
        assert (ctx.ciphertext_residues(out[k]) == want).all(), k
    assert ctx.ciphertext_scale(out[0]) == scale and out[0].limbs == 1
    z = ctx.decrypt_slots(sk, out[0])
    x = o.query_slots(v)
    assert np.abs(z - npcheb.chebval(x, c)).max() < 1e-5


def test_sharded_membership_equals_single(run):
    """Membership under sharding (bench.py, P > 1): each rank's EvalAddMany of its comparison
    ciphertexts, then hd_membership of the partial sums on rank 0 = hd_membership of all."""
    c = hd.chebyshev_coefficients(0.5, 13)
    cmp = run.ctx.compare(run.evk, run.outs, c)
    whole = run.ctx.membership(run.evk, cmp)
    parts = [run.ctx.eval_add_many(cmp[:2]), run.ctx.eval_add_many(cmp[2:])]
    sharded = run.ctx.membership(run.evk, parts)
    torch.cuda.synchronize()
    assert (run.ctx.ciphertext_residues(sharded) == run.ctx.ciphertext_residues(whole)).all()


@pytest.mark.parametrize("n", [1, 2, 3])
def test_compare_low_degrees_bit_exact(run, n):
    """Degenerate Paterson-Stockmeyer shapes (n = 1: d1 = 1, a single scalar product; n = 2, 3)
    on the scan outputs: bit-exact vs the oracle; a constant series is rejected."""
    c = np.array([0.25, -0.5, 0.75, 0.125][: n + 1])
    cmp = run.ctx.compare(run.evk, run.outs, c)
    torch.cuda.synchronize()
    for got, ref in zip(cmp, run.ref_outs):
        want, scale = run.o.cheb_compare(ref, D45, c, run.rlk)
        assert (run.ctx.ciphertext_residues(got) == want).all()
        assert run.ctx.ciphertext_scale(got) == scale
    with pytest.raises(hd.HDError) as e:
        run.ctx.compare(run.evk, run.outs, np.array([1.0, 0.0, 0.0]))
    assert e.value.code == -1


@pytest.mark.slow
def test_membership_at_bench_configuration():
    """`bench.py --scenario membership --packing flat` configuration (2^16 ring, 2^20 x 512, L = 7,
    n1 = 128, 32 aggregates compared in one batch to 2 limbs): every slot of the membership ciphertext
    decrypts to the sum over all 2^20 vectors of the Chebyshev series of their cosine (a
    property that holds at any size; the ciphertext bits are pinned on the smaller configs)."""
    cfg = dataclasses.replace(CONFIGS["C4"], limbs=7)   # membership keeps 2 limbs for its sum (R29)
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    steps = sorted(set(int(s) for s in ctx.rotation_steps(cfg.dim, cfg.n1, packing="flat"))
                   | set(int(s) for s in ctx.membership_steps()))
    sk, evk = ctx.keygen(np.array(steps, np.int32))
    ctx.relin_keygen(sk, evk)
    db = ctx.enroll(db_vecs, cfg.n1, packing="flat")
    outs = ctx.query(evk, db, ctx.encrypt_query(sk, q, ENC_SEED_BASE))
    c = hd.chebyshev_coefficients(0.5, 13)
    cmp = ctx.compare(evk, outs, c, out_limbs=2)
    mem = ctx.membership(evk, cmp)
    torch.cuda.synchronize()
    assert len(cmp) == 32 and cmp[0].limbs == 2 and mem.limbs == 2
    z = ctx.decrypt_slots(sk, mem)
    cos = _cos(db_vecs, q)
    pad = len(cmp) * ctx.ns - cfg.num_vectors
    total = npcheb.chebval(cos, c).sum() + pad * npcheb.chebval(0.0, c)
    assert np.abs(z - total).max() < 1e-3 * max(1.0, abs(total))
    # identification on a sampled aggregate: slot v of comparison a = chebval(cos of vector a M N + v)
    a = 13
    zs = ctx.decrypt_slots(sk, cmp[a])
    assert np.abs(zs - npcheb.chebval(cos[a * ctx.ns:(a + 1) * ctx.ns], c)).max() < 1e-5



def test_compare_to_two_limbs_bit_exact(run):
    """hd_compare_ex with out_limbs = 2 (the membership headroom, R29): degree 5 from 5 limbs,
    bit-exact vs the oracle; a request the levels cannot meet is HD_E_LEVEL."""
    c = hd.chebyshev_coefficients(0.5, 5)
    cmp = run.ctx.compare(run.evk, run.outs, c, out_limbs=2)
    torch.cuda.synchronize()
    for got, ref in zip(cmp, run.ref_outs):
        want, scale = run.o.cheb_compare(ref, D45, c, run.rlk, out_limbs=2)
        assert got.limbs == 2 and (run.ctx.ciphertext_residues(got) == want).all()
        assert run.ctx.ciphertext_scale(got) == scale
    with pytest.raises(hd.HDError) as e:
        run.ctx.compare(run.evk, run.outs, hd.chebyshev_coefficients(0.5, 13), out_limbs=2)
    assert e.value.code == -6



@pytest.mark.slow
def test_membership_at_bench_configuration_scaled_count():
    """The bench's membership at L = 6: the client scales the series by 2^-8 so the 2^20-slot sum
    stays below q_0 / 2 at one limb (R29); the decrypted total times 2^8 is the count."""
    cfg = dataclasses.replace(CONFIGS["C4"], limbs=6)
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    steps = sorted(set(int(s) for s in ctx.rotation_steps(cfg.dim, cfg.n1, packing="flat"))
                   | set(int(s) for s in ctx.membership_steps()))
    sk, evk = ctx.keygen(np.array(steps, np.int32))
    ctx.relin_keygen(sk, evk)
    db = ctx.enroll(db_vecs, cfg.n1, packing="flat")
    outs = ctx.query(evk, db, ctx.encrypt_query(sk, q, ENC_SEED_BASE))
    c = hd.chebyshev_coefficients(0.5, 13)
    mem = ctx.membership(evk, ctx.compare(evk, outs, c * 2.0 ** -8))
    torch.cuda.synchronize()
    assert mem.limbs == 1
    z = ctx.decrypt_slots(sk, mem) * 2.0 ** 8
    cos = _cos(db_vecs, q)
    total = npcheb.chebval(cos, c).sum() + (len(outs) * ctx.ns - cfg.num_vectors) * npcheb.chebval(0.0, c)
    assert np.abs(z - total).max() < 1e-3 * max(1.0, abs(total))


def test_online_aggregated_membership_accuracy(run):
    """Online aggregation (R30, Alg. online-aggr) with the paper's query rescaling
    (P:L2463-2490): the client encrypts q / f_G, f_G = 1 + (G - 1) 2 / sqrt(l), the server scans
    the summed diagonals and compares against delta / f_G.  Every slot of the comparison decodes
    to the Chebyshev series at S[j] / f_G, S[j] = the sum of that slot's cosines over the G
    aggregates (plaintext, float64), which stays inside [-1, 1] (where the series is valid), and
    the membership total is the series summed over every slot.  (How well a degree-13 step
    separates S / f_G around delta / f_G is the paper's false-positive caveat.)"""
    ctx, cfg = run.ctx, run.cfg
    G = len(run.outs)
    f = 1.0 + (G - 1) * 2.0 / np.sqrt(cfg.dim)
    agg = ctx.database_aggregate(run.db)
    qct = ctx.encrypt_query(run.sk, run.q, ENC_SEED_BASE + 7, msg_scale=1.0 / f)
    out = ctx.query(run.evk, agg, qct)
    assert len(out) == 1
    delta = 0.5
    c = hd.chebyshev_coefficients(delta / f, 13)
    cmp = ctx.compare(run.evk, out, c)
    mem = ctx.membership(run.evk, cmp)
    torch.cuda.synchronize()
    # plaintext aggregated score per slot: slot j of aggregate a holds vector a ns + j (flat)
    S = np.zeros(ctx.ns)
    for a in range(G):
        v0, v1 = a * ctx.ns, min(cfg.num_vectors, (a + 1) * ctx.ns)
        S[: v1 - v0] += run.cos[v0:v1]
    assert np.abs(S / f).max() <= 1.0  # the rescaled input stays in the series' interval
    slots = ctx.decrypt_slots(run.sk, cmp[0])
    assert np.abs(slots - npcheb.chebval(S / f, c)).max() < 1e-4
    total = float(ctx.decrypt_slots(run.sk, mem)[0])
    want = float(npcheb.chebval(S / f, c).sum())
    assert abs(total - want) < 1e-3 * max(1.0, abs(want)), (total, want)
