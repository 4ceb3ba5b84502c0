B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 $B > gpurun_out/r3k_kara.log 2>&1; python tools/bsum.py gpurun_out/r3k_kara.log
HD_PACK_D=0 timeout 300 $B > gpurun_out/r3k_nopack.log 2>&1; python tools/bsum.py gpurun_out/r3k_nopack.log
HD_MAC_COMPUTE_ONLY=1 timeout 300 $B --no-check > gpurun_out/r3k_co.log 2>&1; python tools/bsum.py gpurun_out/r3k_co.log
timeout 300 $B --packing flat > gpurun_out/r3k_flat.log 2>&1; python tools/bsum.py gpurun_out/r3k_flat.log
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_flat.py tests/test_gpu_split.py tests/test_gpu_batch.py -q -x > gpurun_out/r3k_pytest.log 2>&1; tail -3 gpurun_out/r3k_pytest.log
