B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0 --no-size-curve --no-check"
run() { tag=$1; shift; env "$@" timeout 300 $B > gpurun_out/r3n_$tag.log 2>&1; python tools/bsum.py gpurun_out/r3n_$tag.log | cut -c1-120; }
run base HD_X=0
run sps4 HD_MAC_SPS=4
run sps4s4 HD_MAC_SPS=4 HD_MAC_STAGES=4
run sps4dry HD_MAC_SPS=4 HD_MAC_TMA_DRY=1
run ag4sps4 HD_MAC_AG=4 HD_MAC_SPS=4
run ag1 HD_MAC_AG=1
