B="python bench.py --no-cpu-baseline --steps 6 --warmup 3 --e2e-steps 0 --no-check"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2z_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2z_$tag.log; }
run b2 HD_X=0 --batch 2
run b4g2 HD_MAC_BATCH=2 --batch 4
run b4 HD_X=0 --batch 4
run b4g1 HD_MAC_BATCH=1 --batch 4
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ -s 6 -c 4 -o gpurun_out/r2z_ntt python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-check > gpurun_out/r2z_ncu.log 2>&1
tail -2 gpurun_out/r2z_ncu.log
