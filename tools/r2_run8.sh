# encrypted-database MAC on the TMA pipeline: parity + A/B
timeout 900 python -m pytest tests/test_gpu_encdb.py tests/test_gpu_flat.py -m gpu -q -x > gpurun_out/r2e8_pytest.log 2>&1; tail -3 gpurun_out/r2e8_pytest.log
B="python bench.py --no-cpu-baseline --steps 6 --warmup 3 --e2e-steps 0 --no-check --db encrypted"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 600 $B "$@" > gpurun_out/r2e8_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2e8_$tag.log; }
run enc_tma HD_X=0
run enc_classic HD_MAC_VARIANT=c
run encflat_tma HD_X=0 --packing flat
run encflat_jt1 HD_MAC_CT_JT=1 --packing flat
run encflat_jt4 HD_MAC_CT_JT=4 HD_MAC_AG=1 --packing flat
run encflat_classic HD_MAC_VARIANT=c --packing flat
