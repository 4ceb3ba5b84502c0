B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 $B > gpurun_out/r4j_k1.log 2>&1; python tools/bsum.py gpurun_out/r4j_k1.log | cut -c1-170
HD_KIP1=0 timeout 300 $B > gpurun_out/r4j_k0.log 2>&1; python tools/bsum.py gpurun_out/r4j_k0.log | cut -c1-170
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_compare.py -q -x -k "toy or c2 or c4_timed or rotate or membership" > gpurun_out/r4j_pytest.log 2>&1; tail -2 gpurun_out/r4j_pytest.log
