B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-size-curve --no-check"
HD_MAC_COMPUTE_ONLY=1 timeout 300 $B > gpurun_out/r3i_co.log 2>&1; python tools/bsum.py gpurun_out/r3i_co.log
HD_MAC_TMA_DRY=1 timeout 300 $B > gpurun_out/r3i_dry.log 2>&1; python tools/bsum.py gpurun_out/r3i_dry.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3i_pytest_gpu.log 2>&1; tail -3 gpurun_out/r3i_pytest_gpu.log
