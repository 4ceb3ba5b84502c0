B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve"
python tools/micro/diag_ntt.py 2>&1 | grep -v "^ \|bad" | grep -v "fwd 1.0 inv 1.0 inv-fwd roundtrip 1.0" ; echo diag-done
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 300 $B > gpurun_out/r3h_split.log 2>&1; python tools/bsum.py gpurun_out/r3h_split.log
timeout 300 $B --packing flat > gpurun_out/r3h_flat.log 2>&1; python tools/bsum.py gpurun_out/r3h_flat.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3h_launch.csv python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check > /dev/null 2>&1
