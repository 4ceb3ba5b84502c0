# MAC with a producer warpgroup + setmaxnreg (launch 112 registers: room for a key-switching CTA)
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2_all or pipelined or large_n1" > gpurun_out/r2w12_pytest.log 2>&1; tail -2 gpurun_out/r2w12_pytest.log
B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-check --no-size-curve"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2w12_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2w12_$tag.log; }
run base HD_X=0
run wgr HD_MAC_WGR=1
run wgrA HD_MAC_WGR=1 HD_PRIO=A
run wgr0 HD_MAC_WGR=1 HD_PRIO=0
run wgrflat HD_MAC_WGR=1 --packing flat
run wgrflatA HD_MAC_WGR=1 HD_PRIO=A --packing flat
