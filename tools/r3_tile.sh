B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 $B > gpurun_out/r4a_def.log 2>&1; python tools/bsum.py gpurun_out/r4a_def.log
HD_MAC_TMA_DRY=1 timeout 300 $B --no-check > gpurun_out/r4a_dry.log 2>&1; python tools/bsum.py gpurun_out/r4a_dry.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "packed or fault or c2 or toy or c4_timed or large_n1" > gpurun_out/r4a_pytest.log 2>&1; tail -2 gpurun_out/r4a_pytest.log
