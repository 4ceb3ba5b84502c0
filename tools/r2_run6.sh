# NTT variants: lazy forward reduction x launch bounds (pytest of the NTT/scan parity first)
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_paperdepth.py -m gpu -q -x -k "not c4 and not c3" > gpurun_out/r2n_pytest.log 2>&1; tail -2 gpurun_out/r2n_pytest.log
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-check"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2n_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2n_$tag.log; }
run lazy HD_X=0
run nolazy HD_LIBHD=paper_2604_00546_b200/libhd_nolazy.so
run lazylb2 HD_LIBHD=paper_2604_00546_b200/libhd_lazylb2.so
run nolazylb2 HD_LIBHD=paper_2604_00546_b200/libhd_nttlb2.so
run lazy_off_rt HD_NTT_LAZY=0
