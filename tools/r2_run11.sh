# combined giant-step sum: parity (replicated, flat, encrypted, split) + bench
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flat.py tests/test_gpu_encdb.py tests/test_gpu_split.py tests/test_gpu_batch.py -m gpu -q -x > gpurun_out/r2g11_pytest.log 2>&1; tail -3 gpurun_out/r2g11_pytest.log
B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-check --no-size-curve"
for t in 1 2; do timeout 300 $B > gpurun_out/r2g11_def$t.log 2>&1; python tools/bsum.py gpurun_out/r2g11_def$t.log; done
timeout 300 $B --packing flat > gpurun_out/r2g11_flat.log 2>&1; python tools/bsum.py gpurun_out/r2g11_flat.log
