# TMA MAC: per-warp arrival, deeper rings (SPS 2, up to 11 stages), AG 2
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0"
run() { tag=$1; shift; env "$@" timeout 300 $B > gpurun_out/r2e_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2e_$tag.log; }
run base HD_MAC_AG=2
run wa HD_MAC_AG=2 HD_MAC_WARP_ARRIVE=1
run sps2 HD_MAC_AG=2 HD_MAC_SPS=2
run sps2wa HD_MAC_AG=2 HD_MAC_SPS=2 HD_MAC_WARP_ARRIVE=1
run ag1sps2 HD_MAC_AG=1 HD_MAC_SPS=2 HD_MAC_WARP_ARRIVE=1
run sps2st6 HD_MAC_AG=2 HD_MAC_SPS=2 HD_MAC_STAGES=6 HD_MAC_WARP_ARRIVE=1
run classic HD_MAC_VARIANT=c
