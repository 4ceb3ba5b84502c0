"""MAC-kernel variant sweep on the bench workload (profiling aid, not a test).

Enrolls the database once, then for each HD_MAC_VARIANT setting ('' = default
streaming kernel, 'g' = generic kernel) runs a few serial queries and prints the per-phase
CUDA-event times.  The variant is read by libhd at every query (getenv), so one
process covers the whole sweep.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_00546_b200 as hd  # noqa: E402
from synth_inputs import CONFIGS, ENC_SEED_BASE, make_dataset  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["", "g"]
os.environ["HD_SERIAL"] = "1"
db_vecs, q, _ = make_dataset(cfg.num_vectors, cfg.dim, cfg.data_seed)
ctx = hd.Context(cfg.log_n, cfg.limbs, seed=1, stream=torch.cuda.current_stream())
sk, evk = ctx.keygen(ctx.rotation_steps(cfg.dim, cfg.n1))
qct = ctx.encrypt_query(sk, q, ENC_SEED_BASE)
db = ctx.enroll(db_vecs, cfg.n1)
outs = None
for v in variants:
    os.environ["HD_MAC_VARIANT"] = v
    for _ in range(2):
        outs = ctx.query(evk, db, qct, outs)
    ctx.query_stats()
    for _ in range(8):
        outs = ctx.query(evk, db, qct, outs)
    ph = ctx.query_stats()
    gbs = cfg.aggregates * cfg.dim * cfg.limbs * (1 << cfg.log_n) * 8 / (ph[1] / 1e3) / 1e9
    print(f"{cfg.name} variant={v or 'default':8s} mac={ph[1]:7.3f} ms ({gbs:6.0f} GB/s)  "
          f"baby={ph[0]:.3f} rescale={ph[2]:.3f} giant={ph[3]:.3f} fold={ph[4]:.3f}", flush=True)
