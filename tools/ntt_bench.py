"""Micro-benchmark of the batched NTT kernels through hd_test_ntt (profiling aid).
Rows are grouped by modulus so each direction is one batched launch pair."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_00546_b200 as hd  # noqa: E402

log_n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 256
# modulus indices cycled over the rows, e.g. "0" (60-bit, integer rows), "1" (45-bit, FP64 rows), "0,1"
mods_arg = [int(x) for x in (sys.argv[3] if len(sys.argv) > 3 else "0").split(",")]
ctx = hd.Context(log_n, 3)
mods, _ = ctx.moduli()
rng = np.random.default_rng(0)
mi = np.array([mods_arg[r % len(mods_arg)] for r in range(rows)], np.uint32)
data = np.stack([rng.integers(0, mods[m], size=1 << log_n, dtype=np.uint64) for m in mi])
for inv in (False, True):
    t0 = time.perf_counter()
    ctx.test_ntt(data, mi, inverse=inv)
    print("inverse" if inv else "forward", time.perf_counter() - t0)
