B="python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_chunks --launch-skip 203 -c 1 -o gpurun_out/r3g_resc_fp64 $B > /dev/null 2>&1
HD_NTT_FP64=0 timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_chunks --launch-skip 203 -c 1 -o gpurun_out/r3g_resc_int $B > /dev/null 2>&1
ls gpurun_out/r3g*
