B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3c_smoke.log 2>&1; tail -1 gpurun_out/r3c_smoke.log
timeout 300 $B > gpurun_out/r3c_fp64.log 2>&1; python tools/bsum.py gpurun_out/r3c_fp64.log
HD_NTT_FP64=0 timeout 300 $B > gpurun_out/r3c_int.log 2>&1; python tools/bsum.py gpurun_out/r3c_int.log
timeout 300 $B --packing flat > gpurun_out/r3c_flat.log 2>&1; python tools/bsum.py gpurun_out/r3c_flat.log
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r3c_pytest_gpu.log 2>&1; tail -3 gpurun_out/r3c_pytest_gpu.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ -c 4 -o gpurun_out/r3c_ntt python tools/ntt_bench.py 16 762 > gpurun_out/r3c_ntt.log 2>&1; tail -1 gpurun_out/r3c_ntt.log
