timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3l_launch.csv python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check > /dev/null 2>&1
python tools/launch_sum.py gpurun_out/r3l_launch.csv
