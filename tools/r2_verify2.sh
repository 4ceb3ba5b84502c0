# Round-2 verification 2: all GPU tests, smoke, the bench lines of every mode, launch list
set -x
mkdir -p gpurun_out/r2v2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2v2/smoke.log 2>&1
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2v2/pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/r2v2/default.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2v2/ref.log 2>&1
timeout 600 python bench.py --packing flat --no-cpu-baseline --no-size-curve > gpurun_out/r2v2/flat.log 2>&1
timeout 900 python bench.py --packing flat --db encrypted --no-cpu-baseline > gpurun_out/r2v2/flat_enc.log 2>&1
timeout 900 python bench.py --db encrypted --no-cpu-baseline > gpurun_out/r2v2/enc.log 2>&1
timeout 900 python bench.py --packing flat --scenario membership --no-cpu-baseline > gpurun_out/r2v2/membership.log 2>&1
timeout 900 python bench.py --scenario identification --no-cpu-baseline > gpurun_out/r2v2/ident.log 2>&1
timeout 900 python bench.py --config C3 --n1 23 --packing flat --db encrypted --scenario membership --no-cpu-baseline > gpurun_out/r2v2/paper_tbe_mem_n23.log 2>&1
timeout 900 python bench.py --config C3 --n1 128 --packing flat --db encrypted --scenario membership --no-cpu-baseline > gpurun_out/r2v2/paper_tbe_mem_n128.log 2>&1
timeout 900 python bench.py --config C3 --profile paper --n1 128 --no-cpu-baseline > gpurun_out/r2v2/paper_depth_C3.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2v2/launches_default.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-check --no-size-curve > gpurun_out/r2v2/ncu_launches.log 2>&1
tail -n 2 gpurun_out/r2v2/smoke.log gpurun_out/r2v2/pytest_gpu.log
python tools/bsum.py gpurun_out/r2v2/*.log
