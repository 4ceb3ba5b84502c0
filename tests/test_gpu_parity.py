"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle, bit-exact on
every RNS residue; decrypted scores vs brute-force cosine within 1e-3 (north star).

Sizes: the toy config C1 (every stage, every aggregate), C2 (2^15 ring, all
aggregates), and the bench configuration C4 (2^16 ring, 2^20 x 512, n1 = 128) in the
bench's timed pipeline mode, on a sampled aggregate the oracle computes one by one.
"""
import numpy as np
import pytest

from synth_inputs import CONFIGS, ENC_SEED_BASE, dataset_rows, make_dataset

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_00546_b200 as hd  # noqa: E402


def _cos(db, q):
    d = db.astype(np.float64)
    qq = q.astype(np.float64)
    return d @ qq / (np.linalg.norm(d, axis=1) * np.linalg.norm(qq))


class Run:
    """One config: GPU objects + oracle objects on identical seeded inputs."""

    def __init__(self, cfg, full_db=True, agg_range=(0, 0)):
        self.cfg = cfg
        self.ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
        self.o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
        self.db_vecs, self.q, self.pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
        self.steps = self.ctx.rotation_steps(cfg.dim, cfg.n1)
        self.sk, self.evk = self.ctx.keygen(self.steps)
        self.qct = self.ctx.encrypt_query(self.sk, self.q, ENC_SEED_BASE)
        self.db = self.ctx.enroll(self.db_vecs, cfg.n1, *agg_range)
        self.outs = self.ctx.query(self.evk, self.db, self.qct)
        torch.cuda.synchronize()
        self._okeys = None

    # oracle side -----------------------------------------------------------------------------
    def oracle_keys(self):
        if self._okeys is None:
            s, s_ntt = self.o.secret_key()
            steps, keys = self.o.keyset(s_ntt, [int(x) for x in self.steps])
            self._okeys = (s_ntt, steps, keys)
        return self._okeys

    def oracle_query_ct(self):
        s_ntt, _, _ = self.oracle_keys()
        z = self.o.query_slots(self.q)
        return self.o.encrypt(s_ntt, self.o.encode(z, 2.0 ** 45, self.cfg.limbs), ENC_SEED_BASE)

    def oracle_D(self, agg):
        cfg = self.cfg
        per = (self.o.ns // cfg.dim // 2) * cfg.dim
        pair = agg - agg % 2   # Alg. enroller_bsgs builds the (ctA, ctB) pair from one temporary
        v0, v1 = pair * per, min(cfg.num_vectors, (pair + 2) * per)
        U = self.o.normalize_rows(self.db_vecs[v0:v1])
        return self.o.enroll_aggregate(U, v0, cfg.num_vectors, cfg.n1, agg)


@pytest.fixture(scope="module")
def toy():
    return Run(CONFIGS["C1"])


def test_moduli_and_roots_match_oracle(toy):
    mods, psi = toy.ctx.moduli()
    assert mods == toy.o.p.moduli
    assert psi == [int(toy.o.p.psi[i]) for i in range(toy.cfg.limbs + 1)]


@pytest.mark.parametrize("log_n", [12, 15, 16])
def test_ntt_bit_exact(log_n):
    ctx = hd.Context(log_n, 3)
    o = oracle.Oracle(log_n, 3)
    rng = np.random.default_rng(log_n)
    rows, mi = [], []
    for l, m in enumerate(o.p.moduli):
        for _ in range(3):
            rows.append(rng.integers(0, m, o.n, dtype=np.uint64))
            mi.append(l)
    rows = np.stack(rows)
    fwd = ctx.test_ntt(rows, mi)
    inv = ctx.test_ntt(rows, mi, inverse=True)
    for r in range(len(rows)):
        assert (fwd[r] == o.ntt(rows[r], mi[r])).all()
        assert (inv[r] == o.ntt(rows[r], mi[r], inverse=True)).all()
    # edge values: 0 and q-1 everywhere
    for l, m in enumerate(o.p.moduli):
        for v in (0, m - 1):
            row = np.full((1, o.n), v, np.uint64)
            assert (ctx.test_ntt(row, [l])[0] == o.ntt(row[0], l)).all()
    # Harvey-lazy inputs in [q, 2q) (the kernels accept [0, 2q); the FP64 rows' bounds, R33,
    # hold up to 4q): the transform of x equals the oracle's transform of x mod q
    for l, m in enumerate(o.p.moduli):
        x = rng.integers(0, m, o.n, dtype=np.uint64)
        lazy = (x + np.uint64(m)).reshape(1, -1)
        for inv in (False, True):
            assert (ctx.test_ntt(lazy, [l], inverse=inv)[0] == o.ntt(x, l, inverse=inv)).all(), (l, inv)
        top = np.full((1, o.n), 2 * m - 1, np.uint64)
        assert (ctx.test_ntt(top, [l], inverse=True)[0] == o.ntt(top[0] - np.uint64(m), l, inverse=True)).all()


def test_keys_bit_exact(toy):
    s_ntt, steps, keys = toy.oracle_keys()
    assert (toy.ctx.secret_key_export(toy.sk) == s_ntt).all()
    gsteps, gkeys = hd.eval_key_residues(toy.ctx, toy.ctx.eval_keys_export(toy.evk))
    assert list(gsteps) == list(steps)
    assert (gkeys == keys).all()


def test_query_encryption_bit_exact(toy):
    assert (toy.ctx.ciphertext_residues(toy.qct) == toy.oracle_query_ct()).all()


def test_rotate_and_rescale_bit_exact(toy):
    s_ntt, steps, keys = toy.oracle_keys()
    qo = toy.oracle_query_ct()
    for st in (1, 5, int(steps[-1])):
        k = keys[list(steps).index(st)]
        got = toy.ctx.ciphertext_residues(toy.ctx.test_rotate(toy.evk, toy.qct, st))
        assert (got == toy.o.rotate(qo, k, st)).all()
    got = toy.ctx.ciphertext_residues(toy.ctx.test_rescale(toy.qct))
    assert (got == toy.o.rescale(qo)).all()


def test_enrollment_bit_exact(toy):
    D = toy.oracle_D(0)
    for k in range(toy.cfg.dim):
        assert (toy.ctx.test_stage(toy.db, 4, 0, k) == D[k]).all(), k


def test_toy_every_stage_bit_exact(toy):
    o, cfg = toy.o, toy.cfg
    s_ntt, steps, keys = toy.oracle_keys()
    r = o.baby_steps(toy.oracle_query_ct(), cfg.n1, steps, keys)
    for i in range(cfg.n1):
        assert (toy.ctx.test_stage(toy.db, 0, 0, i) == r[i]).all(), f"r[{i}]"
    D = toy.oracle_D(0)
    jmin, jmax = o.giant_range(cfg.dim, cfg.n1)
    for j in range(jmin, jmax + 1):
        S = o.giant_sum(r, cfg.n1, cfg.dim, D, j)
        assert (toy.ctx.test_stage(toy.db, 1, 0, j) == S).all(), f"S_{j}"
        assert (toy.ctx.test_stage(toy.db, 2, 0, j) == o.rescale(S)).all(), f"S'_{j}"
    out, y = o.scan_aggregate(r, cfg.n1, cfg.dim, D, steps, keys, want_y=True)
    assert (toy.ctx.test_stage(toy.db, 3, 0, 0) == y).all()
    assert (toy.ctx.ciphertext_residues(toy.outs[0]) == out).all()


def test_toy_scores(toy):
    sc = toy.ctx.decrypt_scores(toy.sk, toy.db.layout, toy.outs)
    cos = _cos(toy.db_vecs, toy.q)
    assert len(sc) == toy.cfg.num_vectors
    assert np.abs(sc - cos).max() < 1e-3
    assert np.abs(sc - cos).max() < 1e-6   # noise budget: a larger error is a bug
    assert sorted(np.argsort(-sc)[:3]) == sorted(toy.pos.tolist())
    # the oracle's decode of the GPU ciphertext agrees
    s_ntt, _, _ = toy.oracle_keys()
    osc = toy.o.decrypt_scores(s_ntt, toy.ctx.ciphertext_residues(toy.outs[0]), toy.cfg.dim, 0,
                               toy.cfg.num_vectors)
    assert np.abs(osc[:len(sc)] - sc).max() < 1e-9


def test_c2_all_aggregates_bit_exact():
    run = Run(CONFIGS["C2"])
    o, cfg = run.o, run.cfg
    s_ntt, steps, keys = run.oracle_keys()
    assert (run.ctx.ciphertext_residues(run.qct) == run.oracle_query_ct()).all()
    r = o.baby_steps(run.oracle_query_ct(), cfg.n1, steps, keys)
    for i in (0, 1, cfg.n1 - 1):
        assert (run.ctx.test_stage(run.db, 0, 0, i) == r[i]).all()
    for a in range(cfg.aggregates):
        D = run.oracle_D(a)
        for k in (0, 1, 255, 256, 511):
            assert (run.ctx.test_stage(run.db, 4, a, k) == D[k]).all()
        out = o.scan_aggregate(r, cfg.n1, cfg.dim, D, steps, keys)
        assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all(), a
    sc = run.ctx.decrypt_scores(run.sk, run.db.layout, run.outs)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:3]) == sorted(run.pos.tolist())


@pytest.mark.parametrize("name", ["C2n128", "C2n256"])
def test_large_n1_bit_exact(name):
    """n1 = 128 / 256 (4 / 2 giant steps): the MAC's carry-save accumulators run at their
    maximum depth and are banked every 128 terms; every output bit-exact vs the oracle."""
    run = Run(CONFIGS[name])
    o, cfg = run.o, run.cfg
    s_ntt, steps, keys = run.oracle_keys()
    r = o.baby_steps(run.oracle_query_ct(), cfg.n1, steps, keys)
    for a in range(cfg.aggregates):
        D = run.oracle_D(a)
        out = o.scan_aggregate(r, cfg.n1, cfg.dim, D, steps, keys)
        assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all(), a
    sc = run.ctx.decrypt_scores(run.sk, run.db.layout, run.outs)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() < 1e-6


@pytest.mark.parametrize("name", ["C1", "C2n256"])
def test_generic_mac_kernel_bit_exact(name, monkeypatch):
    """The generic 128-bit MAC kernel (any n1, partial giant-step ranges; forced here
    with HD_MAC_VARIANT=g) gives the oracle's bits, like the streaming kernel."""
    monkeypatch.setenv("HD_MAC_VARIANT", "g")
    run = Run(CONFIGS[name])
    o, cfg = run.o, run.cfg
    s_ntt, steps, keys = run.oracle_keys()
    r = o.baby_steps(run.oracle_query_ct(), cfg.n1, steps, keys)
    a = cfg.aggregates - 1
    D = run.oracle_D(a)
    out = o.scan_aggregate(r, cfg.n1, cfg.dim, D, steps, keys)
    assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all()


def test_pipelined_queries_match_serial(monkeypatch):
    """Back-to-back queries on the two-stream pipeline (S double-buffered, outputs reused
    in place) give exactly the serial results, for alternating query ciphertexts."""
    cfg = CONFIGS["C1"]
    run = Run(cfg)
    q2 = run.ctx.encrypt_query(run.sk, run.q[::-1].copy(), ENC_SEED_BASE + 1)
    monkeypatch.setenv("HD_SERIAL", "1")
    ref1 = [run.ctx.ciphertext_residues(o) for o in run.ctx.query(run.evk, run.db, run.qct)]
    ref2 = [run.ctx.ciphertext_residues(o) for o in run.ctx.query(run.evk, run.db, q2)]
    monkeypatch.setenv("HD_SERIAL", "0")
    # six queries enqueued back to back (no host sync in between), fresh outputs each
    results = [run.ctx.query(run.evk, run.db, run.qct if it % 2 == 0 else q2) for it in range(6)]
    for it, outs in enumerate(results):
        want = ref1 if it % 2 == 0 else ref2
        got = [run.ctx.ciphertext_residues(o) for o in outs]
        assert all((g == w).all() for g, w in zip(got, want)), it
    # and in place: the same output handles reused by consecutive queries
    outs = None
    for it in range(4):
        outs = run.ctx.query(run.evk, run.db, run.qct if it % 2 == 0 else q2, outs)
    assert all((run.ctx.ciphertext_residues(o) == w).all() for o, w in zip(outs, ref2))


def test_streamed_host_queries_match_serial(monkeypatch):
    """The end-to-end pattern of bench.py: host query bytes imported in place into two
    alternating ciphertexts (upload stream, ordered after the previous query's baby steps),
    outputs reused in place and downloaded asynchronously -- every downloaded result equals
    the serial one, although nothing synchronises the host between steps."""
    cfg = CONFIGS["C1"]
    run = Run(cfg)
    ctx = run.ctx
    qs = [run.qct, ctx.encrypt_query(run.sk, run.q[::-1].copy(), ENC_SEED_BASE + 1)]
    monkeypatch.setenv("HD_SERIAL", "1")
    refs = [[ctx.ciphertext_residues(o) for o in ctx.query(run.evk, run.db, qq)] for qq in qs]
    monkeypatch.setenv("HD_SERIAL", "0")
    blobs = [torch.from_numpy(ctx.ciphertext_export(qq)).pin_memory() for qq in qs]
    qin = [ctx.ciphertext_import(blobs[0].numpy()), ctx.ciphertext_import(blobs[0].numpy())]
    sz = ctx.ciphertext_export_async(run.outs[0], None)
    steps = 6
    host = torch.empty(steps * len(run.outs) * sz, dtype=torch.uint8, pin_memory=True)
    outs = None
    for k in range(steps):
        ctx.ciphertext_import_into(qin[k % 2], blobs[k % 2].data_ptr(), blobs[k % 2].numel(), on_device=False)
        outs = ctx.query(run.evk, run.db, qin[k % 2], outs)
        for i, o in enumerate(outs):
            ctx.ciphertext_export_async(o, (host.data_ptr() + (k * len(outs) + i) * sz, sz))
    ctx.synchronize()
    buf = host.numpy()
    for k in range(steps):
        for i in range(len(outs)):
            off = (k * len(outs) + i) * sz
            got = buf[off + 64:off + sz].view(np.uint64).reshape(2, -1, ctx.n)
            assert (got == refs[k % 2][i]).all(), (k, i)


@pytest.mark.slow
def test_c4_timed_pipeline_full_size(monkeypatch):
    """The bench's timed mode at its full size (2^16 ring, 2^20 x 512, n1 = 128, all 64
    aggregates on one GPU), exactly as bench.py runs it: back-to-back hd_query calls on the
    two-stream pipeline (S double-buffered, outputs reused in place, no host sync between
    steps) over two alternating query ciphertexts, every step's outputs downloaded
    asynchronously (R24 path at full level).  Every output of every step equals the serial
    (HD_SERIAL=1, one stream) result bit for bit; a sampled aggregate of the serial result
    equals the oracle's (or_scan_aggregate_hoisted, R23) bit for bit; and the decrypted
    scores of both queries are within the noise budget (1e-6, north star 1e-3)
    with the planted matches on top."""
    cfg = CONFIGS["C4"]
    run = Run(cfg)
    ctx, o = run.ctx, run.o
    q2v = run.q[::-1].copy()
    qs = [run.qct, ctx.encrypt_query(run.sk, q2v, ENC_SEED_BASE + 1)]
    monkeypatch.setenv("HD_SERIAL", "1")
    refs = []
    for qq in qs:
        outs = ctx.query(run.evk, run.db, qq)
        refs.append([ctx.ciphertext_residues(x) for x in outs])
    monkeypatch.setenv("HD_SERIAL", "0")
    A = len(refs[0])
    sz = ctx.ciphertext_export_async(run.outs[0], None)
    steps = 4
    host = torch.empty(steps * A * sz, dtype=torch.uint8, pin_memory=True)
    outs = run.outs
    torch.cuda.synchronize()
    for k in range(steps):
        outs = ctx.query(run.evk, run.db, qs[k % 2], outs)
        for i, x in enumerate(outs):
            ctx.ciphertext_export_async(x, (host.data_ptr() + (k * A + i) * sz, sz))
    ctx.synchronize()
    buf = host.numpy()
    for k in range(steps):
        for i in range(A):
            off = (k * A + i) * sz
            got = buf[off + 64:off + sz].view(np.uint64).reshape(2, -1, ctx.n)
            assert (got == refs[k % 2][i]).all(), (k, i)
    # the oracle on a sampled aggregate (serial result of query 1); the database's baby-step
    # workspace holds the last query's r, so query 1 runs once more before it is read
    monkeypatch.setenv("HD_SERIAL", "1")
    ctx.query(run.evk, run.db, qs[0], outs)
    torch.cuda.synchronize()
    s_ntt, steps_, keys = run.oracle_keys()
    r = o.baby_steps(run.oracle_query_ct(), cfg.n1, steps_, keys)
    assert (ctx.test_stage(run.db, 0, 0, cfg.n1 - 1) == r[-1]).all()
    a = 37
    out = o.scan_aggregate(r, cfg.n1, cfg.dim, run.oracle_D(a), steps_, keys)
    assert (refs[0][a] == out).all()
    # scores of both queries, from the last two pipelined steps' downloads
    for k, qv in ((steps - 2, run.q), (steps - 1, q2v)):
        cts = [ctx.ciphertext_import(buf[(k * A + i) * sz:(k * A + i + 1) * sz].copy()) for i in range(A)]
        sc = ctx.decrypt_scores(run.sk, run.db.layout, cts)
        err = float(np.abs(sc - _cos(run.db_vecs, qv)).max())
        print(f"C4 step {k}: max |score - cos| = {err:.3e}")
        assert err < 1e-6
    sc = ctx.decrypt_scores(run.sk, run.db.layout, [ctx.ciphertext_import(buf[((steps - 2) * A + i) * sz:
                                                                               ((steps - 2) * A + i + 1) * sz].copy())
                                                    for i in range(A)])
    assert sorted(np.argsort(-sc)[:3]) == sorted(run.pos.tolist())


def test_sharding_invariance_and_partial_aggregates():
    """out_a is bit-identical whatever aggregate range a rank enrolls (P = 1, 2, 3 shards),
    including an odd A with a partial last aggregate (K not a multiple of N)."""
    from synth_inputs import Config
    cfg = Config("shard", 11, 16, 1500, 4, index=9)   # ns = 1024, N = 16, M = 64, G = 94, A = 3
    full = Run(cfg)
    assert cfg.aggregates == 3
    for rng_ in ((0, 1), (1, 3), (2, 3)):
        db = full.ctx.enroll(full.db_vecs, cfg.n1, *rng_)
        outs = full.ctx.query(full.evk, db, full.qct)
        for i, a in enumerate(range(*rng_)):
            assert (full.ctx.ciphertext_residues(outs[i]) == full.ctx.ciphertext_residues(full.outs[a])).all()
    s_ntt, steps, keys = full.oracle_keys()
    r = full.o.baby_steps(full.oracle_query_ct(), cfg.n1, steps, keys)
    D = full.oracle_D(2)
    assert (full.ctx.ciphertext_residues(full.outs[2]) ==
            full.o.scan_aggregate(r, cfg.n1, cfg.dim, D, steps, keys)).all()
    sc = full.ctx.decrypt_scores(full.sk, full.db.layout, full.outs)
    assert len(sc) == cfg.num_vectors
    assert np.abs(sc - _cos(full.db_vecs, full.q)).max() < 1e-6


def test_n1_equals_N_and_reused_outputs():
    from synth_inputs import Config
    cfg = Config("diag", 12, 64, 300, 64, index=10)   # n1 = N: plain diagonal method, no giant rotation
    run = Run(cfg)
    s_ntt, steps, keys = run.oracle_keys()
    r = run.o.baby_steps(run.oracle_query_ct(), cfg.n1, steps, keys)
    out = run.o.scan_aggregate(r, cfg.n1, cfg.dim, run.oracle_D(0), steps, keys)
    assert (run.ctx.ciphertext_residues(run.outs[0]) == out).all()
    # a second query into the same output handles (in place) gives the same bits
    again = run.ctx.query(run.evk, run.db, run.qct, outs=run.outs)
    assert again[0] is run.outs[0]
    assert (run.ctx.ciphertext_residues(again[0]) == out).all()


def test_errors():
    ctx = hd.Context(12, 3)
    v = np.ones((100, 64), np.float32)
    v[17] = 0
    with pytest.raises(hd.HDError) as e:
        ctx.enroll(v, 8)
    assert e.value.code == hd.HD_E_ZERO_VECTOR
    with pytest.raises(hd.HDError) as e:
        ctx.enroll(np.ones((10, 48), np.float32), 8)         # not a power of two
    assert e.value.code == hd.HD_E_LAYOUT
    with pytest.raises(hd.HDError) as e:
        ctx.enroll(np.ones((10, 2048), np.float32), 8)       # numSlots % 2N != 0
    assert e.value.code == hd.HD_E_LAYOUT
    sk, evk = ctx.keygen(ctx.rotation_steps(64, 8)[:-1])    # drop the fold key
    db = ctx.enroll(np.ones((100, 64), np.float32), 8)
    qct = ctx.encrypt_query(sk, np.ones(64, np.float32), 5)
    with pytest.raises(hd.HDError) as e:
        ctx.query(evk, db, qct)
    assert e.value.code == hd.HD_E_MISSING_KEY and "1984" in str(e.value)
    import ctypes as C
    big = hd.Context(16, 3)
    out = C.c_void_p()
    few = np.ones((4, 512), np.float32)   # the capacity check precedes any read of the rows
    rc = hd.load().hd_enroll(big.h, few.ctypes.data_as(C.c_void_p), 1 << 26, 512, 64, 0, 0, C.byref(out))
    assert rc == hd.HD_E_CAPACITY and not out.value          # 2^26 vectors: ~3.3 TB of diagonals


def test_level_reduced_async_export():
    """hd_ciphertext_export_async at 1 limb (R24): the exported residues are limb 0 of
    the outputs bit for bit, they decrypt to the cosine scores, and a query issued right
    after the export (no host sync) does not overwrite the outputs before the copies ran."""
    run = Run(CONFIGS["C1"])
    ctx, cfg = run.ctx, run.cfg
    full = [ctx.ciphertext_residues(o) for o in run.outs]
    sz = ctx.ciphertext_export_async(run.outs[0], None, nlimbs=1)
    assert sz == 64 + 2 * ctx.n * 8
    host = torch.empty(len(run.outs) * sz, dtype=torch.uint8, pin_memory=True)
    for i, o in enumerate(run.outs):
        ctx.ciphertext_export_async(o, (host.data_ptr() + i * sz, sz), nlimbs=1)
    rng = np.random.default_rng(5)
    q2 = rng.standard_normal(cfg.dim).astype(np.float32)
    ctx.query(run.evk, run.db, ctx.encrypt_query(run.sk, q2, ENC_SEED_BASE + 1), run.outs)  # overwrites outs
    ctx.synchronize()
    buf = host.numpy()
    cts = []
    for i in range(len(run.outs)):
        blob = buf[i * sz:(i + 1) * sz].copy()
        got = blob[64:].view(np.uint64).reshape(2, 1, ctx.n)
        assert (got[:, 0] == full[i][:, 0]).all(), i
        cts.append(ctx.ciphertext_import(blob))
    sc = ctx.decrypt_scores(run.sk, run.db.layout, cts)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() < 1e-6
    with pytest.raises(hd.HDError):
        ctx.ciphertext_export_async(run.outs[0], None, nlimbs=cfg.limbs)  # outputs have L-1 limbs


def test_fault_injection_is_detected():
    """The parity checks catch a single flipped residue bit: flipping one bit of one diagonal
    word of aggregate 1 (C2, two aggregates) changes that aggregate's output ciphertext (now
    unequal to the oracle's) and leaves aggregate 0 bit-exact; flipping it back restores parity.
    The flipped coefficient is an NTT-domain residue, so after decryption the error spreads over
    every slot of the block: the score check fails too."""
    run = Run(CONFIGS["C2"])
    o, cfg, ctx = run.o, run.cfg, run.ctx
    s_ntt, steps, keys = run.oracle_keys()
    r = o.baby_steps(run.oracle_query_ct(), cfg.n1, steps, keys)
    want = [o.scan_aggregate(r, cfg.n1, cfg.dim, run.oracle_D(a), steps, keys) for a in range(cfg.aggregates)]
    assert all((ctx.ciphertext_residues(run.outs[a]) == want[a]).all() for a in range(cfg.aggregates))
    ctx.test_inject(run.db, 1, 37, 12345, 1 << 20)
    outs = ctx.query(run.evk, run.db, run.qct)
    assert (ctx.ciphertext_residues(outs[0]) == want[0]).all()
    assert not (ctx.ciphertext_residues(outs[1]) == want[1]).all()
    sc = ctx.decrypt_scores(run.sk, run.db.layout, outs)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() > 1e-3
    ctx.test_inject(run.db, 1, 37, 12345, 1 << 20)  # restore
    outs = ctx.query(run.evk, run.db, run.qct, outs)
    assert all((ctx.ciphertext_residues(outs[a]) == want[a]).all() for a in range(cfg.aggregates))


def test_packed_and_unpacked_diagonals_bit_exact(monkeypatch):
    """Packed plaintext diagonals (R34: the 45-bit limbs in 6 bytes, split at bit 31) are the
    default where the TMA MAC serves the layout; HD_PACK_D=0 at enrollment keeps u64 words.
    Both layouts give the oracle's bits on every aggregate, hd_test_stage returns the same
    residues from either, and the reported diagonal size is 20 n / 24 n bytes at L = 3."""
    cfg = CONFIGS["C2"]
    packed = Run(cfg)
    monkeypatch.setenv("HD_PACK_D", "0")
    plain = Run(cfg)
    monkeypatch.delenv("HD_PACK_D")
    n = 1 << cfg.log_n
    assert packed.db.diagonal_bytes == (20 * n, True)
    assert plain.db.diagonal_bytes == (24 * n, False)
    o = packed.o
    s_ntt, steps, keys = packed.oracle_keys()
    r = o.baby_steps(packed.oracle_query_ct(), cfg.n1, steps, keys)
    for a in range(cfg.aggregates):
        want = o.scan_aggregate(r, cfg.n1, cfg.dim, packed.oracle_D(a), steps, keys)
        for run in (packed, plain):
            assert (run.ctx.ciphertext_residues(run.outs[a]) == want).all(), a
    for k in (0, 7, cfg.dim - 1):
        dp = packed.ctx.test_stage(packed.db, 4, 1, k)
        du = plain.ctx.test_stage(plain.db, 4, 1, k)
        assert (dp == du).all()
        assert (dp.reshape(cfg.limbs, n) == packed.oracle_D(1)[k]).all()
