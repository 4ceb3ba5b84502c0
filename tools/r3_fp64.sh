B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3b_smoke.log 2>&1; tail -1 gpurun_out/r3b_smoke.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "ntt or toy or c2" > gpurun_out/r3b_pytest_quick.log 2>&1; tail -2 gpurun_out/r3b_pytest_quick.log
timeout 300 $B > gpurun_out/r3b_fp64.log 2>&1; python tools/bsum.py gpurun_out/r3b_fp64.log
HD_NTT_FP64=0 timeout 300 $B > gpurun_out/r3b_int.log 2>&1; python tools/bsum.py gpurun_out/r3b_int.log
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r3b_pytest_gpu.log 2>&1; tail -3 gpurun_out/r3b_pytest_gpu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ -c 4 -o gpurun_out/r3b_ntt python tools/ntt_bench.py 16 762 > gpurun_out/r3b_ntt.log 2>&1; tail -1 gpurun_out/r3b_ntt.log
