B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-check --no-size-curve"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2w13_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2w13_$tag.log; }
run base HD_X=0
run wgrco HD_MAC_WGR=1 HD_CARVEOUT=1
run wgrcoA HD_MAC_WGR=1 HD_CARVEOUT=1 HD_PRIO=A
run wgrco0 HD_MAC_WGR=1 HD_CARVEOUT=1 HD_PRIO=0
