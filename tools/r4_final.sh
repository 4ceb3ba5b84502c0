nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r4g_smoke.log 2>&1; tail -1 gpurun_out/r4g_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r4g_pytest_gpu.log 2>&1; tail -3 gpurun_out/r4g_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r4g_default.json 2> gpurun_out/r4g_default.err; python tools/bsum.py gpurun_out/r4g_default.json
