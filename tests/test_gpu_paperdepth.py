"""GPU parity at the paper-depth key-switching profile (SURVEY 8(d) "secondary"; R31: L = 12
limbs, alpha = 4 limbs per digit, K_sp = 4 special primes), through the C ABI,
bit-exact against the CPU oracle (oracle pinned in tests/test_oracle_paperdepth.py).

* toy ring (C1 workload at L = 12): keys, the query, every stage of the scan, all outputs;
  rotations and rescales at every level the scan uses;
* C3 at P = 1 (ring 2^15, 2^17 x 512, n1 = 16, 16 aggregates, L = 12): a sampled aggregate
  bit-exact, every score within the noise budget, the planted matches on top.
"""
import numpy as np
import pytest

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


class Run:
    def __init__(self, cfg):
        self.cfg = cfg
        prof = dict(num_special=cfg.special, digit_limbs=cfg.digit_limbs)
        self.ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1, **prof)
        self.o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1, K_sp=cfg.special, alpha=cfg.digit_limbs)
        self.db_vecs, self.q, self.pos = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
        self.steps = self.ctx.rotation_steps(cfg.dim, cfg.n1)
        self.sk, self.evk = self.ctx.keygen(self.steps)
        self.qct = self.ctx.encrypt_query(self.sk, self.q, ENC_SEED_BASE)
        self.db = self.ctx.enroll(self.db_vecs, cfg.n1)
        self.outs = self.ctx.query(self.evk, self.db, self.qct)
        torch.cuda.synchronize()
        self._ok = None

    def okeys(self):
        if self._ok is None:
            _, s_ntt = self.o.secret_key()
            steps, keys = self.o.keyset(s_ntt, [int(x) for x in self.steps])
            self._ok = (s_ntt, steps, keys)
        return self._ok

    def oquery(self):
        s_ntt = self.okeys()[0]
        return self.o.encrypt(s_ntt, self.o.encode(self.o.query_slots(self.q), D45, self.cfg.limbs), ENC_SEED_BASE)

    def oD(self, agg):
        cfg = self.cfg
        per = (self.o.ns // cfg.dim // 2) * cfg.dim
        pair = agg - agg % 2
        v0, v1 = pair * per, min(cfg.num_vectors, (pair + 2) * per)
        return self.o.enroll_aggregate(self.o.normalize_rows(self.db_vecs[v0:v1]), v0, cfg.num_vectors, cfg.n1, agg)


@pytest.fixture(scope="module")
def toy():
    return Run(CONFIGS["C1p"])


def test_profile_moduli_and_keys(toy):
    mods, psi = toy.ctx.moduli()
    assert mods == toy.o.p.moduli and len(mods) == 16
    s_ntt, steps, keys = toy.okeys()
    assert (toy.ctx.secret_key_export(toy.sk) == s_ntt).all()
    gsteps, gkeys = hd.eval_key_residues(toy.ctx, toy.ctx.eval_keys_export(toy.evk))
    assert list(gsteps) == list(steps)
    assert gkeys.shape == (len(steps), 3, 2, 16, toy.ctx.n)
    assert (gkeys == keys).all()
    assert (toy.ctx.ciphertext_residues(toy.qct) == toy.oquery()).all()


def test_rotations_and_rescale_every_level(toy):
    s_ntt, steps, keys = toy.okeys()
    qo = toy.oquery()
    ct_g, ct_o = toy.qct, qo
    for level in (12, 11, 9, 5, 4, 2):
        while ct_o.shape[1] > level:  # walk down by rescaling on both sides
            ct_o = toy.o.rescale(ct_o)
            ct_g = toy.ctx.test_rescale(ct_g)
            assert (toy.ctx.ciphertext_residues(ct_g) == ct_o).all(), ct_o.shape
        for st in (1, 7, int(steps[-1])):
            k = keys[list(steps).index(st)]
            got = toy.ctx.ciphertext_residues(toy.ctx.test_rotate(toy.evk, ct_g, st))
            assert (got == toy.o.rotate(ct_o, k, st)).all(), (level, st)


def test_toy_every_stage_and_scores(toy):
    o, cfg = toy.o, toy.cfg
    s_ntt, steps, keys = toy.okeys()
    r = o.baby_steps(toy.oquery(), cfg.n1, steps, keys)
    for i in range(cfg.n1):
        assert (toy.ctx.test_stage(toy.db, 0, 0, i) == r[i]).all(), f"r[{i}]"
    D = toy.oD(0)
    jmin, jmax = o.giant_range(cfg.dim, cfg.n1)
    for j in range(jmin, jmax + 1):
        S = o.giant_sum(r, cfg.n1, cfg.dim, D, j)
        assert (toy.ctx.test_stage(toy.db, 1, 0, j) == S).all(), f"S_{j}"
        assert (toy.ctx.test_stage(toy.db, 2, 0, j) == o.rescale(S)).all(), f"S'_{j}"
    out = o.scan_aggregate(r, cfg.n1, cfg.dim, D, steps, keys)
    assert (toy.ctx.ciphertext_residues(toy.outs[0]) == out).all()
    sc = toy.ctx.decrypt_scores(toy.sk, toy.db.layout, toy.outs)
    assert np.abs(sc - _cos(toy.db_vecs, toy.q)).max() < 1e-6
    assert sorted(np.argsort(-sc)[:3]) == sorted(toy.pos.tolist())


def test_relinearisation_refused_at_general_profile(toy):
    with pytest.raises(hd.HDError) as ei:
        toy.ctx.compare(toy.evk, toy.outs, hd.chebyshev_coefficients(0.5, 13))
    assert ei.value.code == hd.HD_E_PARAMS


@pytest.mark.slow
def test_c3_paper_depth_sampled_aggregate():
    run = Run(CONFIGS["C3p"])
    o, cfg = run.o, run.cfg
    s_ntt, steps, keys = run.okeys()
    r = o.baby_steps(run.oquery(), cfg.n1, steps, keys)
    assert (run.ctx.test_stage(run.db, 0, 0, cfg.n1 - 1) == r[-1]).all()
    a = 11
    out = o.scan_aggregate(r, cfg.n1, cfg.dim, run.oD(a), steps, keys)
    assert (run.ctx.ciphertext_residues(run.outs[a]) == out).all()
    sc = run.ctx.decrypt_scores(run.sk, run.db.layout, run.outs)
    err = float(np.abs(sc - _cos(run.db_vecs, run.q)).max())
    print(f"C3 paper depth: max |score - cos| = {err:.3e}")
    assert err < 1e-6
    assert sorted(np.argsort(-sc)[:3]) == sorted(run.pos.tolist())
