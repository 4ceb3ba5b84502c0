# carve-out (max shared for the key-switching kernels so they can sit beside the MAC CTA) x priority
# x NTT CTA size; KIP with batched digit loads (default build)
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-check --no-size-curve"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2c10_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2c10_$tag.log; }
run base HD_X=0
run co HD_CARVEOUT=1
run coA HD_CARVEOUT=1 HD_PRIO=A
run co128 HD_CARVEOUT=1 HD_LIBHD=paper_2604_00546_b200/libhd_ntt128.so
run co128A HD_CARVEOUT=1 HD_PRIO=A HD_LIBHD=paper_2604_00546_b200/libhd_ntt128.so
run co128_0 HD_CARVEOUT=1 HD_PRIO=0 HD_LIBHD=paper_2604_00546_b200/libhd_ntt128.so
