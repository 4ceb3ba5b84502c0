"""GPU parity of the encrypted-database mode (NEXT-1, R26): the CUDA path through the C ABI
vs the CPU oracle, bit-exact on every residue (public key, relinearisation key, encrypted
diagonals, degree-2 giant sums, relinearised sums, outputs); decrypted scores vs
brute-force cosine within 1e-6 (north-star tolerance 1e-3)."""
import numpy as np
import pytest

from synth_inputs import CONFIGS, ENC_SEED_BASE, make_dataset

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_00546_b200 as hd  # noqa: E402

DB_SEED = 4242


def _cos(db, q):
    d = db.astype(np.float64)
    qq = q.astype(np.float64)
    return d @ qq / (np.linalg.norm(d, axis=1) * np.linalg.norm(qq))


class EncRun:
    def __init__(self, cfg):
        self.cfg = cfg
        self.ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
        self.o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
        self.db_vecs, self.q, self.pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
        self.steps = self.ctx.rotation_steps(cfg.dim, cfg.n1)
        self.sk, self.evk = self.ctx.keygen(self.steps)
        self.ctx.relin_keygen(self.sk, self.evk)
        self.pk = self.ctx.public_keygen(self.sk)
        self.qct = self.ctx.encrypt_query(self.sk, self.q, ENC_SEED_BASE)
        self.db = self.ctx.enroll_encrypted(self.pk, self.db_vecs, cfg.n1, DB_SEED)
        self.outs = self.ctx.query(self.evk, self.db, self.qct)
        torch.cuda.synchronize()
        s, self.s_ntt = self.o.secret_key()
        self.ok_steps, self.ok_keys = self.o.keyset(self.s_ntt, [int(x) for x in self.steps])
        self.opk = self.o.public_key(self.s_ntt)
        self.orlk = self.o.relin_key(self.s_ntt)

    def oracle_r(self):
        z = self.o.query_slots(self.q)
        qct = self.o.encrypt(self.s_ntt, self.o.encode(z, 2.0 ** 45, self.cfg.limbs), ENC_SEED_BASE)
        return self.o.baby_steps(qct, self.cfg.n1, self.ok_steps, self.ok_keys)

    def oracle_Dct(self, agg):
        cfg = self.cfg
        per = (self.o.ns // cfg.dim // 2) * cfg.dim
        pair = agg - agg % 2   # Alg. enroller_bsgs builds the (ctA, ctB) pair from one temporary
        v0, v1 = pair * per, min(cfg.num_vectors, (pair + 2) * per)
        U = self.o.normalize_rows(self.db_vecs[v0:v1])
        return self.o.enroll_aggregate_encrypted(U, v0, cfg.num_vectors, cfg.n1, agg, self.opk, DB_SEED)


@pytest.fixture(scope="module")
def toy():
    return EncRun(CONFIGS["C1"])


def test_public_and_relinearisation_keys_bit_exact(toy):
    assert (toy.ctx.public_key_export(toy.pk) == toy.opk).all()
    steps, keys = hd.eval_key_residues(toy.ctx, toy.ctx.eval_keys_export(toy.evk))
    assert steps[-1] == 0  # the relinearisation key's reserved step
    assert (keys[-1] == toy.orlk).all()
    assert (keys[0] == toy.ok_keys[0]).all()  # rotation keys unchanged by the shared key kernels


def test_encrypted_diagonals_sums_and_outputs_bit_exact(toy):
    cfg, o, ctx = toy.cfg, toy.o, toy.ctx
    r = toy.oracle_r()
    Dct = toy.oracle_Dct(0)
    for k in (0, 1, cfg.dim // 2, cfg.dim - 1):
        assert (ctx.test_stage(toy.db, 4, 0, k) == Dct[k]).all(), k
    jmin, jmax = o.giant_range(cfg.dim, cfg.n1)
    for j in (jmin, 0, jmax):
        S3 = o.giant_sum_ct(r, cfg.n1, cfg.dim, Dct, j)
        got = ctx.test_stage(toy.db, 1, 0, j)
        assert (got == S3).all(), j                              # degree-2 sum as accumulated
        # relinearised and rescaled in one rounding = Relinearize then Rescale (R29)
        assert (ctx.test_stage(toy.db, 2, 0, j) == o.rescale(o.relinearize(S3, toy.orlk))).all(), j
    out, y = o.scan_aggregate_ct(r, cfg.n1, cfg.dim, Dct, toy.ok_steps, toy.ok_keys, toy.orlk, want_y=True)
    assert (ctx.test_stage(toy.db, 3, 0, 0) == y).all()
    assert (ctx.ciphertext_residues(toy.outs[0]) == out).all()


def test_encrypted_scores(toy):
    sc = toy.ctx.decrypt_scores(toy.sk, toy.db.layout, toy.outs)
    cos = _cos(toy.db_vecs, toy.q)
    assert np.abs(sc - cos).max() < 1e-6
    assert sorted(np.argsort(-sc)[:len(toy.pos)]) == sorted(toy.pos.tolist())


def test_encrypted_c2_all_aggregates_bit_exact():
    run = EncRun(CONFIGS["C2"])
    cfg, o = run.cfg, run.o
    r = run.oracle_r()
    for a in range(cfg.aggregates):
        out = o.scan_aggregate_ct(r, cfg.n1, cfg.dim, run.oracle_Dct(a), run.ok_steps, run.ok_keys, run.orlk)
        assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all(), a
    sc = run.ctx.decrypt_scores(run.sk, run.db.layout, run.outs)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() < 1e-6
    # the encrypted diagonals are stored packed (R34: both polynomials, 45-bit limbs in 6
    # bytes) and hd_test_stage returns the oracle's residues from them
    n = 1 << cfg.log_n
    assert run.db.diagonal_bytes == (2 * 20 * n, True)
    for k in (0, cfg.dim - 1):
        assert (run.ctx.test_stage(run.db, 4, 1, k) == run.oracle_Dct(1)[k]).all()


def test_missing_relinearisation_key_and_public_key_roundtrip(toy):
    ctx = toy.ctx
    _, evk_norelin = ctx.keygen(toy.steps)
    with pytest.raises(hd.HDError) as ei:
        ctx.query(evk_norelin, toy.db, toy.qct)
    assert ei.value.code == -5  # HD_E_MISSING_KEY
    pk2 = ctx.public_key_import(ctx.public_key_export(toy.pk))
    assert (ctx.public_key_export(pk2) == toy.opk).all()
    bad = toy.opk.copy()
    bad[0, 0, 0] = np.uint64(2 ** 63)
    with pytest.raises(hd.HDError):
        ctx.public_key_import(bad)


def test_generic_degree2_mac_bit_exact(monkeypatch):
    """The general degree-2 MAC (partial giant-step ranges, any n1; forced with
    HD_MAC_VARIANT=g) gives the same bits as the streaming one and the oracle."""
    monkeypatch.setenv("HD_MAC_VARIANT", "g")
    run = EncRun(CONFIGS["C1"])
    cfg, o = run.cfg, run.o
    out = o.scan_aggregate_ct(run.oracle_r(), cfg.n1, cfg.dim, run.oracle_Dct(0), run.ok_steps, run.ok_keys,
                              run.orlk)
    assert (run.ctx.ciphertext_residues(run.outs[0]) == out).all()


@pytest.mark.slow
def test_encrypted_c4_bench_config_sampled_aggregate():
    """`bench.py --db encrypted` configuration (2^16 ring, 2^20 x 512 encrypted diagonals,
    103 GB on one GPU): bit-exact on a sampled aggregate, scores everywhere vs cosine."""
    run = EncRun(CONFIGS["C4"])
    cfg, o = run.cfg, run.o
    a = 50
    out = o.scan_aggregate_ct(run.oracle_r(), cfg.n1, cfg.dim, run.oracle_Dct(a), run.ok_steps, run.ok_keys,
                              run.orlk)
    assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all()
    sc = run.ctx.decrypt_scores(run.sk, run.db.layout, run.outs)
    assert np.abs(sc - _cos(run.db_vecs, run.q)).max() < 1e-3
    assert sorted(np.argsort(-sc)[:3]) == sorted(run.pos.tolist())
