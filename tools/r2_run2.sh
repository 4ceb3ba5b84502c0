# pytest -m gpu (context refcount fix), stream-priority A/B, paper-depth n1 sweep
set -x
mkdir -p gpurun_out/r2w
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2w/pytest_gpu.log 2>&1
tail -n 3 gpurun_out/r2w/pytest_gpu.log
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-check"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2w/$tag.log 2>&1; python tools/bsum.py gpurun_out/r2w/$tag.log; }
run prioB HD_X=0
run prioA HD_PRIO=A
run prio0 HD_PRIO=0
run n64 HD_X=0 --n1 64
run n256 HD_X=0 --n1 256
run pap64 HD_X=0 --config C3 --profile paper --n1 64
run pap128 HD_X=0 --config C3 --profile paper --n1 128
