B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 $B --packing flat --db encrypted > gpurun_out/r4e_fe.log 2>&1; python tools/bsum.py gpurun_out/r4e_fe.log | cut -c1-140
timeout 300 $B --db encrypted > gpurun_out/r4e_e.log 2>&1; python tools/bsum.py gpurun_out/r4e_e.log | cut -c1-140
timeout 300 $B --packing flat_tbs --db encrypted > gpurun_out/r4e_tbs.log 2>&1; python tools/bsum.py gpurun_out/r4e_tbs.log | cut -c1-140
timeout 1500 python -m pytest tests/test_gpu_encdb.py tests/test_gpu_split.py tests/test_gpu_compare.py tests/test_gpu_flat.py -q -x > gpurun_out/r4e_pytest.log 2>&1; tail -3 gpurun_out/r4e_pytest.log
