B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 $B > gpurun_out/r4c_def.log 2>&1; python tools/bsum.py gpurun_out/r4c_def.log
timeout 300 $B --batch 2 > gpurun_out/r4c_b2.log 2>&1; python tools/bsum.py gpurun_out/r4c_b2.log | cut -c1-60
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r4c_launches.csv python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check > /dev/null 2>&1
python tools/launch_sum.py gpurun_out/r4c_launches.csv
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -q -x -k "toy or c2 or c4_timed or batch or large_n1" > gpurun_out/r4c_pytest.log 2>&1; tail -2 gpurun_out/r4c_pytest.log
