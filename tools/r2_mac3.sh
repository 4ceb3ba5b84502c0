# TMA MAC: AG=4 inline producer vs AG=2 producer warp vs the LDG kernel; batch 4; parity
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0"
run() { tag=$1; shift; env "$@" timeout 300 $B > gpurun_out/r2d_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2d_$tag.log; }
run ag4 HD_MAC_AG=4
run ag2 HD_MAC_AG=2
run ag4sep HD_MAC_AG=4 HD_MAC_INLINE=0
run classic HD_MAC_VARIANT=c
HD_MAC_AG=4 timeout 300 python bench.py --no-cpu-baseline --steps 4 --warmup 2 --e2e-steps 0 --batch 4 > gpurun_out/r2d_b4.log 2>&1; python tools/bsum.py gpurun_out/r2d_b4.log
HD_MAC_AG=4 timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --packing flat > gpurun_out/r2d_flat.log 2>&1; python tools/bsum.py gpurun_out/r2d_flat.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mac_tma -c 1 -o gpurun_out/r2d_mac_tma python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/r2d_ncu.log 2>&1
timeout 900 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_flat.py -m gpu -q -x > gpurun_out/r2d_pytest.log 2>&1
tail -3 gpurun_out/r2d_pytest.log
