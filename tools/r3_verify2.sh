python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3w_smoke.log 2>&1; tail -1 gpurun_out/r3w_smoke.log
timeout 900 python -m pytest tests/test_gpu_encdb.py -q -x > gpurun_out/r3w_pytest_enc.log 2>&1; tail -2 gpurun_out/r3w_pytest_enc.log
timeout 900 python bench.py > gpurun_out/r3w_default.json 2> gpurun_out/r3w_default.err; python tools/bsum.py gpurun_out/r3w_default.json
timeout 600 python bench.py --packing flat --no-cpu-baseline --no-size-curve > gpurun_out/r3w_flat.json 2>&1; python tools/bsum.py gpurun_out/r3w_flat.json
timeout 600 python bench.py --db encrypted --no-cpu-baseline --no-size-curve > gpurun_out/r3w_enc.json 2>&1; python tools/bsum.py gpurun_out/r3w_enc.json
timeout 600 python bench.py --packing flat --db encrypted --no-cpu-baseline --no-size-curve > gpurun_out/r3w_flatenc.json 2>&1; python tools/bsum.py gpurun_out/r3w_flatenc.json
timeout 600 python bench.py --packing flat --scenario membership --no-cpu-baseline --no-size-curve > gpurun_out/r3w_mem.json 2>&1; python tools/bsum.py gpurun_out/r3w_mem.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3w_ref.json 2>&1
B1="python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3w_launches.csv $B1 > /dev/null 2>&1
python tools/launch_sum.py gpurun_out/r3w_launches.csv
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:mac_ -c 1 --csv --log-file gpurun_out/r3w_mac_traffic.csv $B1 > /dev/null 2>&1
du -sh gpurun_out
