B="python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3d_launch_fp64.csv $B > gpurun_out/r3d_l1.log 2>&1
HD_NTT_FP64=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3d_launch_int.csv $B > gpurun_out/r3d_l0.log 2>&1
tail -2 gpurun_out/r3d_l1.log gpurun_out/r3d_l0.log
