"""bench.py's N > 1 path, end to end on one CUDA device (gloo, both ranks on cuda:0 via
HD_BENCH_ONE_GPU=1): sharded enrollment, the StepExchange broadcast / gather of 1-limb result
exports, max-over-ranks timing and the rank-0 score check over every shard.  A functional test
of the multi-GPU code, not a measurement (the line's timing shares one GPU)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("extra", [["--config", "C2"],
                                   ["--config", "C2", "--split-baby"],
                                   ["--config", "C3", "--packing", "flat", "--scenario", "membership"]])
def test_two_ranks_on_one_gpu(extra):
    env = dict(os.environ, HD_BENCH_ONE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + len(extra)), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--no-cpu-baseline", *extra]
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1  # rank 0 prints once
    d = lines[0]
    assert d["n_gpus"] == 2 and d["config"]["parallelism"] == "aggregate-shard x2"
    assert d["split_baby"] == ("--split-baby" in extra)
    if "--scenario" not in extra:  # the scan: every score of both shards checked on rank 0
        assert d["check"]["ok"] and d["check"]["scores_checked"] == 1 << 14
