B1="python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mac_tma -c 1 -o gpurun_out/r3y_mac $B1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kip_giant1 -c 1 -o gpurun_out/r3y_kipg $B1 > /dev/null 2>&1
du -sh gpurun_out/*
