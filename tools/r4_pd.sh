timeout 900 python -m pytest tests/test_gpu_paperdepth.py tests/test_gpu_hardening.py -q > gpurun_out/r4h_pytest.log 2>&1; tail -2 gpurun_out/r4h_pytest.log
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-size-curve --profile paper"
timeout 300 $B --config C3 --n1 128 > gpurun_out/r4h_c3.log 2>&1; python tools/bsum.py gpurun_out/r4h_c3.log | cut -c1-150
timeout 300 $B > gpurun_out/r4h_c4.log 2>&1; python tools/bsum.py gpurun_out/r4h_c4.log | cut -c1-150
