# NTT CTA size (128 threads: one can sit beside a MAC CTA) x stream priority; chunk twiddles in smem
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-check --no-size-curve"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2q_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2q_$tag.log; }
run base HD_X=0
run base_prioA HD_PRIO=A
run n128 HD_LIBHD=paper_2604_00546_b200/libhd_ntt128.so
run n128_prioA HD_LIBHD=paper_2604_00546_b200/libhd_ntt128.so HD_PRIO=A
run n128_prio0 HD_LIBHD=paper_2604_00546_b200/libhd_ntt128.so HD_PRIO=0
run twsmem HD_LIBHD=paper_2604_00546_b200/libhd_twsmem.so
run base2 HD_X=0
