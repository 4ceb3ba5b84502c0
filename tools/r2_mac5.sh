B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0"
run() { tag=$1; shift; env "$@" timeout 300 $B > gpurun_out/r2f_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2f_$tag.log; }
run compute HD_MAC_AG=2 HD_MAC_COMPUTE_ONLY=1
run dry HD_MAC_AG=2 HD_MAC_TMA_DRY=1
run ag1s8 HD_MAC_AG=1 HD_MAC_SPS=8
run ag1s8dry HD_MAC_AG=1 HD_MAC_SPS=8 HD_MAC_TMA_DRY=1
run ag1s4 HD_MAC_AG=1
