"""Per-rank compute time of a P-way sharded C4 scan, simulated on one GPU (no NCCL).

For P in {1, 2, 4, 8}: one database handle holding A/P aggregates; time (CUDA events) of
  (a) hd_query: every rank recomputes all n1 - 1 baby steps, and
  (b) hd_baby_steps on a 1/P slice + hd_query_baby from a full r buffer (the all-gather of r,
      384 MiB at n1 = 128, is NOT included: ~0.4 ms over NVLink 5 at P = 8).
Prints one JSON line per P.  Usage: python tools/shard_sim.py [--config C4] [--iters 10]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_00546_b200 as hd  # noqa: E402
from synth_inputs import CONFIGS, ENC_SEED_BASE, dataset_rows, make_dataset  # noqa: E402


def timed(fn, iters, stream):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    stream = torch.cuda.current_stream()
    ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1, stream=stream)
    _, q, _ = make_dataset(16, cfg.dim, cfg.data_seed)
    sk, evk = ctx.keygen(ctx.rotation_steps(cfg.dim, cfg.n1))
    qct = ctx.encrypt_query(sk, q, ENC_SEED_BASE)
    per = (cfg.num_slots // cfg.dim // 2) * cfg.dim
    A = -(-cfg.num_vectors // per)
    ct_l = 2 * cfg.limbs * (1 << cfg.log_n)
    r = torch.empty(cfg.n1 * ct_l, dtype=torch.int64, device="cuda")
    for P in (1, 2, 4, 8):
        a1 = A // P
        v1 = min(cfg.num_vectors, a1 * per)
        rows = dataset_rows(cfg.num_vectors, cfg.dim, cfg.data_seed, 0, v1)
        db = ctx.enroll(rows, cfg.n1, 0, a1)
        del rows
        outs = [None]

        def full():
            outs[0] = ctx.query(evk, db, qct, outs[0])

        chunk = -(-cfg.n1 // P)

        def split():
            ctx.baby_steps(evk, db, qct, 0, min(cfg.n1, chunk), r.data_ptr())
            outs[0] = ctx.query_baby(evk, db, r.data_ptr(), outs[0])

        ctx.baby_steps(evk, db, qct, 0, cfg.n1, r.data_ptr())  # r complete (stands in for the all-gather)
        t_full = timed(full, args.iters, stream)
        t_split = timed(split, args.iters, stream)
        print(json.dumps({"P": P, "aggregates_per_rank": a1, "ms_full_baby": t_full, "ms_split_baby": t_split,
                          "speedup_vs_P1_full": None}), flush=True)
        del db
        torch.cuda.synchronize()


if __name__ == "__main__":
    main()
