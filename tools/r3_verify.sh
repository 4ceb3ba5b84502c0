set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r3v_smoke.log 2>&1; tail -1 gpurun_out/r3v_smoke.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "packed or ntt or fault or c4_timed" > gpurun_out/r3v_pytest_new.log 2>&1; tail -2 gpurun_out/r3v_pytest_new.log
timeout 900 python bench.py > gpurun_out/r3v_default.json 2> gpurun_out/r3v_default.err; python tools/bsum.py gpurun_out/r3v_default.json
timeout 600 python bench.py --packing flat --no-cpu-baseline --no-size-curve > gpurun_out/r3v_flat.json 2>&1; python tools/bsum.py gpurun_out/r3v_flat.json
timeout 600 python bench.py --db encrypted --no-cpu-baseline --no-size-curve > gpurun_out/r3v_enc.json 2>&1; python tools/bsum.py gpurun_out/r3v_enc.json
timeout 600 python bench.py --packing flat --scenario membership --no-cpu-baseline --no-size-curve > gpurun_out/r3v_mem.json 2>&1; python tools/bsum.py gpurun_out/r3v_mem.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3v_ref.json 2>&1; tail -c 300 gpurun_out/r3v_ref.json
B1="python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3v_launches.csv $B1 > /dev/null 2>&1
python tools/launch_sum.py gpurun_out/r3v_launches.csv
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mac_tma -c 1 -o gpurun_out/r3v_mac $B1 > /dev/null 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:mac_ -c 1 --csv --log-file gpurun_out/r3v_mac_traffic.csv $B1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kip_giant1 -c 1 -o gpurun_out/r3v_kipg $B1 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ -c 4 -o gpurun_out/r3v_ntt_int python tools/ntt_bench.py 16 762 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:ntt_ -c 4 -o gpurun_out/r3v_ntt_fp python tools/ntt_bench.py 16 762 1 > /dev/null 2>&1
ls gpurun_out/r3v*
