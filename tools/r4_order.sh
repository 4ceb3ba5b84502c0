B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
for o in 0 1; do
HD_MAC_ORDER=$o timeout 300 $B > gpurun_out/r4o_o$o.log 2>&1; python tools/bsum.py gpurun_out/r4o_o$o.log | cut -c1-110
HD_MAC_ORDER=$o timeout 300 $B --packing flat > gpurun_out/r4o_f$o.log 2>&1; python tools/bsum.py gpurun_out/r4o_f$o.log | cut -c1-110
HD_MAC_ORDER=$o timeout 300 $B --packing flat --db encrypted > gpurun_out/r4o_fe$o.log 2>&1; python tools/bsum.py gpurun_out/r4o_fe$o.log | cut -c1-110
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_encdb.py tests/test_gpu_batch.py -q -x -k "toy or c2 or c4_timed or packed or large_n1 or batch or encrypted" > gpurun_out/r4o_pytest.log 2>&1; tail -2 gpurun_out/r4o_pytest.log
