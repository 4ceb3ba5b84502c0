# MAC register cap (room for one key-switching CTA per SM) x stream priority
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-check"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2x_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2x_$tag.log; }
run base HD_X=0
run capB HD_MAC_REGCAP=1
run capA HD_MAC_REGCAP=1 HD_PRIO=A
run cap0 HD_MAC_REGCAP=1 HD_PRIO=0
run capflatB HD_MAC_REGCAP=1 --packing flat
run flatB HD_X=0 --packing flat
