"""GPU parity of the split baby steps (hd_baby_steps / hd_query_baby).  With the
database sharded over P GPUs each rank computes a slice of the n1 - 1 baby rotations and an
all-gather assembles r; here the slices (ragged, as for P = 3) are written into one device
buffer on one GPU, and the scan from that buffer must equal hd_query bit for bit, also for
aggregate shards of the database."""
import numpy as np
import pytest

from synth_inputs import CONFIGS, ENC_SEED_BASE, make_dataset

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2604_00546_b200 as hd  # noqa: E402


@pytest.mark.parametrize("name,packing", [("C2", "replicated"), ("C1", "flat")])
def test_split_baby_steps_equal_hd_query(name, packing):
    cfg = CONFIGS[name]
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    sk, evk = ctx.keygen(ctx.rotation_steps(cfg.dim, cfg.n1, packing=packing))
    qct = ctx.encrypt_query(sk, q, ENC_SEED_BASE)
    db_ref = ctx.enroll(db_vecs, cfg.n1, packing=packing)
    ref = [ctx.ciphertext_residues(o) for o in ctx.query(evk, db_ref, qct)]
    db = ctx.enroll(db_vecs, cfg.n1, packing=packing)  # fresh handle: nothing left from hd_query
    n1, L, n = cfg.n1, cfg.limbs, 1 << cfg.log_n
    r = torch.zeros(n1 * 2 * L * n, dtype=torch.int64, device="cuda")
    bounds = [0, n1 // 3, (2 * n1) // 3 + 1, n1]            # three ragged "rank" slices
    for i0, i1 in zip(bounds[:-1], bounds[1:]):
        ctx.baby_steps(evk, db, qct, i0, i1, r.data_ptr())
    outs = ctx.query_baby(evk, db, r.data_ptr())
    torch.cuda.synchronize()
    for a, o in enumerate(outs):
        assert (ctx.ciphertext_residues(o) == ref[a]).all(), a
    # aggregate shards (one database handle per "rank") scanned from the same gathered r
    A = db.num_local
    if A > 1:
        for a0, a1 in ((0, A // 2), (A // 2, A)):
            part = ctx.enroll(db_vecs, cfg.n1, a0, a1, packing=packing)
            got = ctx.query_baby(evk, part, r.data_ptr())
            torch.cuda.synchronize()
            for i, o in enumerate(got):
                assert (ctx.ciphertext_residues(o) == ref[a0 + i]).all(), (a0, i)
    with pytest.raises(hd.HDError):
        ctx.baby_steps(evk, db, qct, 0, n1 + 1, r.data_ptr())


@pytest.mark.parametrize("name,packing,encrypted", [("C2", "replicated", False), ("C1big", "flat", True)])
def test_online_aggregation_bit_exact(name, packing, encrypted):
    """Online DB aggregation (NEXT-4, Alg. online-aggr): the aggregated handle's
    diagonals equal the oracle's residue-wise sum of every aggregate's diagonals, and its scan
    output equals the oracle's scan of that sum, bit for bit."""
    import dataclasses

    import oracle
    from synth_inputs import Config
    cfg = CONFIGS["C2"] if name == "C2" else Config("agg", 12, 64, 5000, 8, index=12)
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1)
    o = oracle.Oracle(cfg.log_n, cfg.limbs, seed=1)
    db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
    steps = ctx.rotation_steps(cfg.dim, cfg.n1, packing=packing)
    sk, evk = ctx.keygen(steps)
    pk = None
    if encrypted:
        ctx.relin_keygen(sk, evk)
        pk = ctx.public_keygen(sk)
    db = ctx.enroll(db_vecs, cfg.n1, packing=packing, pk=pk, enc_seed=7)
    agg = ctx.database_aggregate(db)
    assert agg.num_local == 1
    out = ctx.query(evk, agg, ctx.encrypt_query(sk, q, ENC_SEED_BASE))
    torch.cuda.synchronize()
    _, s_ntt = o.secret_key()
    st, keys = o.keyset(s_ntt, [int(x) for x in steps])
    A = db.num_local
    U = o.normalize_rows(db_vecs)
    if packing == "flat":
        per = o.ns
        opk, orlk = o.public_key(s_ntt), o.relin_key(s_ntt)
        Ds = [o.enroll_aggregate_flat_encrypted(U[a * per:(a + 1) * per], a * per, cfg.num_vectors, cfg.n1, a, opk, 7)
              for a in range(A)]
    else:
        per = (o.ns // cfg.dim // 2) * cfg.dim
        Ds = [o.enroll_aggregate(U[(a - a % 2) * per:(a - a % 2 + 2) * per], (a - a % 2) * per, cfg.num_vectors,
                                 cfg.n1, a) for a in range(A)]
    Dsum = o.aggregate_diagonals(Ds)
    for k in (0, cfg.dim - 1):
        assert (ctx.test_stage(agg, 4, 0, k) == Dsum[k]).all(), k
    qct = o.encrypt(s_ntt, o.encode(o.query_slots(q), 2.0 ** 45, cfg.limbs), ENC_SEED_BASE)
    r = o.baby_steps(qct, cfg.n1, st, keys)
    if packing == "flat":
        ref = o.scan_aggregate_flat_ct(r, cfg.n1, cfg.dim, Dsum, st, keys, orlk)
    else:
        ref = o.scan_aggregate(r, cfg.n1, cfg.dim, Dsum, st, keys)
    assert (ctx.ciphertext_residues(out[0]) == ref).all()
