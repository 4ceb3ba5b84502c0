nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r5_smoke.log 2>&1; tail -1 gpurun_out/r5_smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r5_pytest_gpu.log 2>&1; tail -3 gpurun_out/r5_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r5_default.json 2> gpurun_out/r5_default.err; python tools/bsum.py gpurun_out/r5_default.json
timeout 600 python bench.py --packing flat --no-cpu-baseline --no-size-curve > gpurun_out/r5_flat.json 2>&1; python tools/bsum.py gpurun_out/r5_flat.json
timeout 600 python bench.py --packing flat --db encrypted --no-cpu-baseline --no-size-curve > gpurun_out/r5_flatenc.json 2>&1; python tools/bsum.py gpurun_out/r5_flatenc.json
timeout 600 python bench.py --db encrypted --no-cpu-baseline --no-size-curve > gpurun_out/r5_enc.json 2>&1; python tools/bsum.py gpurun_out/r5_enc.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r5_ref.json 2>&1
B1="python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r5_launches.csv $B1 > /dev/null 2>&1
python tools/launch_sum.py gpurun_out/r5_launches.csv
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:mac_ -c 1 --csv --log-file gpurun_out/r5_mac_traffic.csv $B1 > /dev/null 2>&1
