"""GPU parity of the flat pre-rotated layout (NEXT-2, R27: BSGS-RTX-TBE): the CUDA path
through the C ABI vs the CPU oracle, bit-exact on every residue (pre-rotated diagonals,
giant-step sums, outputs); decrypted scores vs brute-force cosine within 1e-6."""
import numpy as np
import pytest

from synth_inputs import CONFIGS, ENC_SEED_BASE, make_dataset

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


class FlatRun:
    def __init__(self, cfg, n1=None):
        self.cfg, self.n1 = cfg, n1 or cfg.n1
        self.ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
        self.o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
        self.db_vecs, self.q, self.pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
        self.steps = self.ctx.rotation_steps(cfg.dim, self.n1, packing="flat")
        self.sk, self.evk = self.ctx.keygen(self.steps)
        self.qct = self.ctx.encrypt_query(self.sk, self.q, ENC_SEED_BASE)
        self.db = self.ctx.enroll(self.db_vecs, self.n1, packing="flat")
        self.outs = self.ctx.query(self.evk, self.db, self.qct)
        torch.cuda.synchronize()
        s, self.s_ntt = self.o.secret_key()
        self.ok_steps, self.ok_keys = self.o.keyset(self.s_ntt, [int(x) for x in self.steps])

    def oracle_r(self):
        z = self.o.query_slots(self.q)
        qct = self.o.encrypt(self.s_ntt, self.o.encode(z, 2.0 ** 45, self.cfg.limbs), ENC_SEED_BASE)
        return self.o.baby_steps(qct, self.n1, self.ok_steps, self.ok_keys)

    def oracle_D(self, agg):
        cfg, per = self.cfg, self.o.ns
        v0, v1 = agg * per, min(cfg.num_vectors, (agg + 1) * per)  # M N = numSlots vectors per ciphertext
        U = self.o.normalize_rows(self.db_vecs[v0:v1])
        return self.o.enroll_aggregate_flat(U, v0, cfg.num_vectors, self.n1, agg)


@pytest.fixture(scope="module")
def toy():
    return FlatRun(CONFIGS["C1"])


def test_flat_layout_and_keys(toy):
    lay = toy.db.layout
    M = toy.ctx.ns // toy.cfg.dim
    assert lay.packing == 1 and lay.groups_per_ct == M and lay.giant_min == 0
    assert lay.giant_max == -(-toy.cfg.dim // toy.n1) - 1
    assert [int(s) for s in toy.steps] == toy.o.rotation_steps_flat(toy.cfg.dim, toy.n1)


def test_flat_every_stage_bit_exact(toy):
    cfg, o, ctx = toy.cfg, toy.o, toy.ctx
    r = toy.oracle_r()
    D = toy.oracle_D(0)
    for k in (0, 1, toy.n1, cfg.dim - 1):
        assert (ctx.test_stage(toy.db, 4, 0, k) == D[k]).all(), k
    for j in range(lay_jmax(toy) + 1):
        assert (ctx.test_stage(toy.db, 1, 0, j) == o.giant_sum_flat(r, toy.n1, cfg.dim, D, j)).all(), j
    out = o.scan_aggregate_flat(r, toy.n1, cfg.dim, D, toy.ok_steps, toy.ok_keys)
    assert (ctx.ciphertext_residues(toy.outs[0]) == out).all()


def lay_jmax(run):
    return run.db.layout.giant_max


def test_flat_scores(toy):
    sc = toy.ctx.decrypt_scores(toy.sk, toy.db.layout, toy.outs)
    assert np.abs(sc - _cos(toy.db_vecs, toy.q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:len(toy.pos)]) == sorted(toy.pos.tolist())


@pytest.mark.parametrize("name,n1", [("C2", 16), ("C2", 23)])
def test_flat_c2_bit_exact(name, n1):
    """All aggregates of C2; n1 = 23 (the paper's CPU choice) leaves a partial last giant step
    and exercises the general MAC kernel."""
    run = FlatRun(CONFIGS[name], n1)
    cfg, o = run.cfg, run.o
    r = run.oracle_r()
    for a in range(run.db.layout.num_aggregates):
        out = o.scan_aggregate_flat(r, run.n1, cfg.dim, run.oracle_D(a), run.ok_steps, run.ok_keys)
        assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all(), a
    sc = run.ctx.decrypt_scores(run.sk, run.db.layout, run.outs)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() < 1e-6


@pytest.mark.parametrize("name,n1", [("C2", 16), ("C1", 12)])
def test_flat_encrypted_database_bit_exact(name, n1):
    """BSGS-RTX-TBE with encrypted diagonals (the paper's GPU setting): pre-rotated flat
    diagonals encrypted under the public key, degree-2 MAC with the flat ranges,
    relinearisation, no fold; every residue equals the oracle's.  n1 = 12 does not divide
    N = 64: full giant steps on the streaming kernel, the partial last one on the general."""
    import dataclasses
    cfg = dataclasses.replace(CONFIGS[name], n1=n1)
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    steps = ctx.rotation_steps(cfg.dim, cfg.n1, packing="flat")
    sk, evk = ctx.keygen(steps)
    ctx.relin_keygen(sk, evk)
    pk = ctx.public_keygen(sk)
    db = ctx.enroll(db_vecs, cfg.n1, packing="flat", pk=pk, enc_seed=99)
    outs = ctx.query(evk, db, ctx.encrypt_query(sk, q, ENC_SEED_BASE))
    s, s_ntt = o.secret_key()
    ok_steps, ok_keys = o.keyset(s_ntt, [int(x) for x in steps])
    opk, orlk = o.public_key(s_ntt), o.relin_key(s_ntt)
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), 2.0 ** 45, cfg.limbs), ENC_SEED_BASE)
    r = o.baby_steps(qct, cfg.n1, ok_steps, ok_keys)
    for a in range(db.layout.num_aggregates):
        v0, v1 = a * o.ns, min(cfg.num_vectors, (a + 1) * o.ns)
        Dct = o.enroll_aggregate_flat_encrypted(o.normalize_rows(db_vecs[v0:v1]), v0, cfg.num_vectors, cfg.n1, a,
                                                opk, 99)
        assert (ctx.test_stage(db, 4, a, cfg.dim - 1) == Dct[-1]).all(), a
        out = o.scan_aggregate_flat_ct(r, cfg.n1, cfg.dim, Dct, ok_steps, ok_keys, orlk)
        assert (ctx.ciphertext_residues(outs[a]) == out).all(), a
    sc = ctx.decrypt_scores(sk, db.layout, outs)
    assert np.abs(sc - _cos(db_vecs, q)).max() < 1e-6


@pytest.mark.slow
def test_flat_c4_bench_config_sampled_aggregate():
    """`bench.py --packing flat` configuration (2^16 ring, 2^20 x 512, n1 = 128, all 32
    aggregates on one GPU): bit-exact on a sampled aggregate, scores everywhere vs cosine."""
    run = FlatRun(CONFIGS["C4"])
    o, cfg = run.o, run.cfg
    r = run.oracle_r()
    a = 21
    out = o.scan_aggregate_flat(r, run.n1, cfg.dim, run.oracle_D(a), run.ok_steps, run.ok_keys)
    assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all()
    sc = run.ctx.decrypt_scores(run.sk, run.db.layout, run.outs)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() < 1e-3
    assert sorted(np.argsort(-sc)[:3]) == sorted(run.pos.tolist())


def test_flat_tbs_server_prerotation_bit_exact():
    """BSGS-RTX-TBS: plain flat diagonals encrypted by the enroller, pre-rotated
    on the GPU with the negative giant-step keys (hd_database_prerotate) -- the stored
    ciphertexts before and after the pre-rotation and the scan outputs equal the oracle's."""
    cfg = CONFIGS["C1"]
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    N, n1 = cfg.dim, cfg.n1
    neg = ctx.prerotation_steps(N, n1)
    assert [int(x) for x in neg] == sorted(ctx.ns - j * n1 for j in range(1, -(-N // n1)))
    steps = np.array(sorted(set(int(x) for x in ctx.rotation_steps(N, n1, packing="flat")) | set(int(x) for x in neg)),
                     np.int32)
    sk, evk = ctx.keygen(steps)
    ctx.relin_keygen(sk, evk)
    pk = ctx.public_keygen(sk)
    db = ctx.enroll(db_vecs, n1, packing="flat_tbs", pk=pk, enc_seed=5)
    qct = ctx.encrypt_query(sk, q, ENC_SEED_BASE)
    with pytest.raises(hd.HDError):
        ctx.query(evk, db, qct)  # not yet pre-rotated
    s, s_ntt = o.secret_key()
    ok_steps, ok_keys = o.keyset(s_ntt, [int(x) for x in steps])
    opk, orlk = o.public_key(s_ntt), o.relin_key(s_ntt)
    D0 = o.enroll_aggregate_flat_tbs(o.normalize_rows(db_vecs), 0, cfg.num_vectors, n1, 0, opk, 5)
    for k in (0, n1, N - 1):
        assert (ctx.test_stage(db, 4, 0, k) == D0[k]).all(), k
    ctx.database_prerotate(evk, db)
    D1 = o.prerotate_tbs(D0, n1, ok_steps, ok_keys)
    for k in (0, n1, 2 * n1 + 3, N - 1):
        assert (ctx.test_stage(db, 4, 0, k) == D1[k]).all(), k
    outs = ctx.query(evk, db, qct)
    r = o.baby_steps(o.encrypt(s_ntt, o.encode(o.query_slots(q), 2.0 ** 45, cfg.limbs), ENC_SEED_BASE), n1, ok_steps,
                     ok_keys)
    out = o.scan_aggregate_flat_ct(r, n1, N, D1, ok_steps, ok_keys, orlk)
    assert (ctx.ciphertext_residues(outs[0]) == out).all()
    sc = ctx.decrypt_scores(sk, db.layout, outs)
    assert np.abs(sc - _cos(db_vecs, q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:len(pos)]) == sorted(pos.tolist())
