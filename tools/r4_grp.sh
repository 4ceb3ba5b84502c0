B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python tools/micro/diag_ntt.py 2>&1 | grep -v "^ \|bad" | grep -v "fwd 1.0 inv 1.0 inv-fwd roundtrip 1.0"; echo diag-done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 $B > gpurun_out/r4k_g.log 2>&1; python tools/bsum.py gpurun_out/r4k_g.log | cut -c1-170
HD_NTT_GROUPED=0 timeout 300 $B > gpurun_out/r4k_ng.log 2>&1; python tools/bsum.py gpurun_out/r4k_ng.log | cut -c1-170
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "ntt or toy or c2 or c4_timed or packed" > gpurun_out/r4k_pytest.log 2>&1; tail -2 gpurun_out/r4k_pytest.log
