set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2a_pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/r2a_default.log 2>&1
tail -n 3 gpurun_out/r2a_smoke.log gpurun_out/r2a_pytest_gpu.log gpurun_out/r2a_default.log
