B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python tools/micro/diag_ntt.py 2>&1 | grep -v "^ \|bad" | grep -v "fwd 1.0 inv 1.0 inv-fwd roundtrip 1.0"; echo diag-done
timeout 300 $B > gpurun_out/r3o_def.log 2>&1; python tools/bsum.py gpurun_out/r3o_def.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r3o_pytest_gpu.log 2>&1; tail -3 gpurun_out/r3o_pytest_gpu.log
