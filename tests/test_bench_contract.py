"""The bench.py contract on CPU: `--impl reference` times the CPU oracle and prints one
JSON line with the keys the driver reads (no GPU needed)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def test_reference_arm_membership_scenario():
    """NEXT-3: the comparison scenarios run at six limbs and name the tail in the metric."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0", "--scenario", "membership"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][0])
    assert "membership" in d["metric"] and d["config"]["limbs"] == 6 and d["value"] > 0
    assert "ChebyshevCompare" in d["cpu_baseline"]["sample"]


def test_planted_positions_match_make_dataset():
    """bench.py's score check regenerates the planted-match positions without the rows."""
    from synth_inputs import make_dataset, planted_positions
    for K, dim, seed in ((256, 64, 260400547), (5000, 64, 7), (1 << 14, 512, 260400548)):
        _, _, pos = make_dataset(K, dim, seed)
        assert (planted_positions(K, dim, seed) == pos).all()


def test_reference_arm_config_equals_ours():
    """The reference arm's config dict is built by the same function as ours (same_config)."""
    import importlib.util
    import os
    spec = importlib.util.spec_from_file_location("bench", os.path.join(os.path.dirname(__file__), "..", "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    import sys
    argv = sys.argv
    try:
        sys.argv = ["bench.py"]
        args = bench.parse()
    finally:
        sys.argv = argv
    cfg = bench.workload_cfg(args)
    assert bench.full_config(args, cfg, 1)["aggregates"] == cfg.aggregates
    assert args.e2e_steps == args.steps
