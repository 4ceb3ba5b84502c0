"""GPU parity of query batching (NEXT-4, hd_query_batch): every output of a batch of Q queries
is bit-identical to hd_query of that query alone (which the other GPU tests pin to the oracle),
and one batch member is checked against the CPU oracle directly.  Covers the default per-query
MAC, the shared-D batched MAC kernel (HD_MAC_BATCH = 2 / 4: groups of 4 / 2 / 1 queries, the
n1 > 128 banking variant), the per-query path for partial giant-step ranges, both packings,
and in-place reuse of the outputs."""
import dataclasses
import os

import numpy as np
import pytest

from synth_inputs import CONFIGS, ENC_SEED_BASE, make_dataset

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2604_00546_b200 as hd  # noqa: E402


def _setup(cfg, n1, packing):
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    sk, evk = ctx.keygen(ctx.rotation_steps(cfg.dim, n1, packing=packing))
    db = ctx.enroll(db_vecs, n1, packing=packing)
    rng = np.random.default_rng(7)
    return ctx, sk, evk, db, db_vecs, q, rng


@pytest.mark.parametrize("name,n1,packing,Q", [
    ("C1", 8, "replicated", 5),     # groups 4 + 1
    ("C1", 8, "flat", 3),           # groups 2 + 1
    ("C1", 12, "replicated", 2),    # n1 does not divide N/2: per-query MAC fallback
    ("C2", 256, "replicated", 4),   # n1 > 128: the banking variant of the batched kernel
])
@pytest.mark.parametrize("group", ["default", "2", "4"])
def test_batch_equals_single_queries(name, n1, packing, Q, group, monkeypatch):
    if group != "default":   # the shared-D batched MAC kernel (HD_MAC_BATCH)
        monkeypatch.setenv("HD_MAC_BATCH", group)
    cfg = CONFIGS[name]
    ctx, sk, evk, db, db_vecs, q, rng = _setup(cfg, n1, packing)
    qs = [q] + [rng.integers(-99, 100, cfg.dim).astype(np.float32) for _ in range(Q - 1)]
    cts = [ctx.encrypt_query(sk, v, ENC_SEED_BASE + i) for i, v in enumerate(qs)]
    outs = ctx.query_batch(evk, db, cts)
    torch.cuda.synchronize()
    got = [[ctx.ciphertext_residues(o) for o in row] for row in outs]
    for i, ct in enumerate(cts):
        single = ctx.query(evk, db, ct)
        torch.cuda.synchronize()
        for a, o in enumerate(single):
            assert (ctx.ciphertext_residues(o) == got[i][a]).all(), (i, a)
    # in place: a second batch into the same outputs (different order) gives the permuted bits
    again = ctx.query_batch(evk, db, cts[::-1], outs=outs)
    torch.cuda.synchronize()
    assert again[0][0] is outs[0][0]
    for i in range(Q):
        for a in range(db.num_local):
            assert (ctx.ciphertext_residues(again[i][a]) == got[Q - 1 - i][a]).all()


def test_batch_member_matches_the_oracle():
    cfg = CONFIGS["C1"]
    ctx, sk, evk, db, db_vecs, q, rng = _setup(cfg, cfg.n1, "replicated")
    q2 = rng.integers(-99, 100, cfg.dim).astype(np.float32)
    cts = [ctx.encrypt_query(sk, q, ENC_SEED_BASE), ctx.encrypt_query(sk, q2, ENC_SEED_BASE + 1)]
    outs = ctx.query_batch(evk, db, cts)
    torch.cuda.synchronize()
    o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
    _, s_ntt = o.secret_key()
    st, keys = o.keyset(s_ntt, [int(s) for s in ctx.rotation_steps(cfg.dim, cfg.n1)])
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q2), 2.0 ** 45, cfg.limbs), ENC_SEED_BASE + 1)
    r = o.baby_steps(qct, cfg.n1, st, keys)
    D = o.enroll_aggregate(o.normalize_rows(db_vecs), 0, cfg.num_vectors, cfg.n1, 0)
    ref = o.scan_aggregate(r, cfg.n1, cfg.dim, D, st, keys)
    assert (ctx.ciphertext_residues(outs[1][0]) == ref).all()
    scores = ctx.decrypt_scores(sk, db.layout, outs[1])
    d = db_vecs.astype(np.float64)
    cos = d @ q2.astype(np.float64) / (np.linalg.norm(d, axis=1) * np.linalg.norm(q2.astype(np.float64)))
    assert np.abs(scores - cos).max() < 1e-6


def test_batch_errors():
    cfg = dataclasses.replace(CONFIGS["C1"])
    ctx, sk, evk, db, db_vecs, q, rng = _setup(cfg, cfg.n1, "replicated")
    ct = ctx.encrypt_query(sk, q, ENC_SEED_BASE)
    with pytest.raises(hd.HDError):
        ctx.query_batch(evk, db, [])
    pk = ctx.public_keygen(sk)
    ctx.relin_keygen(sk, evk)
    edb = ctx.enroll(db_vecs, cfg.n1, pk=pk, enc_seed=3)
    with pytest.raises(hd.HDError) as e:
        ctx.query_batch(evk, edb, [ct, ct])
    assert e.value.code == -1


@pytest.mark.slow
def test_c4_batch_matches_single_queries():
    """The bench configuration (2^16 ring, 2^20 x 512, n1 = 128, 64 aggregates): a batch of
    two queries through the batched MAC equals hd_query of each, on every aggregate."""
    cfg = CONFIGS["C4"]
    ctx, sk, evk, db, db_vecs, q, rng = _setup(cfg, cfg.n1, "replicated")
    q2 = rng.integers(-99, 100, cfg.dim).astype(np.float32)
    cts = [ctx.encrypt_query(sk, q, ENC_SEED_BASE), ctx.encrypt_query(sk, q2, ENC_SEED_BASE + 1)]
    os.environ["HD_MAC_BATCH"] = "2"   # the shared-D kernel at the bench configuration
    try:
        outs = ctx.query_batch(evk, db, cts)
        torch.cuda.synchronize()
    finally:
        os.environ.pop("HD_MAC_BATCH")
    got = [[ctx.ciphertext_residues(o) for o in row] for row in outs]
    for i, ct in enumerate(cts):
        single = ctx.query(evk, db, ct)
        torch.cuda.synchronize()
        assert len(single) == 64
        for a, o in enumerate(single):
            assert (ctx.ciphertext_residues(o) == got[i][a]).all(), (i, a)
