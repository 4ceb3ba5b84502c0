timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ -c 2 -o gpurun_out/r2p_ntt python tools/ntt_bench.py 16 1024 > gpurun_out/r2p_ntt.log 2>&1
tail -3 gpurun_out/r2p_ntt.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kip_kernel -c 1 -o gpurun_out/r2p_kip python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-check > gpurun_out/r2p_kip.log 2>&1
tail -3 gpurun_out/r2p_kip.log
