set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3a_smoke.log 2>&1
tail -2 gpurun_out/r3a_smoke.log
timeout 300 python bench.py --no-cpu-baseline --steps 20 --warmup 5 --no-size-curve > gpurun_out/r3a_default.log 2>&1
python tools/bsum.py gpurun_out/r3a_default.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ -c 4 -o gpurun_out/r3a_ntt python tools/ntt_bench.py 16 762 > gpurun_out/r3a_ntt.log 2>&1
tail -3 gpurun_out/r3a_ntt.log
