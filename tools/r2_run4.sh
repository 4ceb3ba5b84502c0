B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-check"
run() { tag=$1; shift; envs=(); while [[ "$1" == *=* ]]; do envs+=("$1"); shift; done; env "${envs[@]}" timeout 300 $B "$@" > gpurun_out/r2y_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2y_$tag.log; }
run ch0 HD_NTT_CHUNK=0
run ch96 HD_NTT_CHUNK=96
run ch48 HD_NTT_CHUNK=48
run ch192 HD_NTT_CHUNK=192
run ch24 HD_NTT_CHUNK=24
