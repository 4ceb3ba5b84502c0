B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0"
run() { tag=$1; shift; env "$@" timeout 300 $B > gpurun_out/r2g_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2g_$tag.log; }
run pf0 HD_MAC_AG=2 HD_MAC_PF=0
run pf4 HD_MAC_AG=2 HD_MAC_PF=4
run pf8 HD_MAC_AG=2 HD_MAC_PF=8
run pf16 HD_MAC_AG=2 HD_MAC_PF=16
run pf32 HD_MAC_AG=2 HD_MAC_PF=32
run s2pf16 HD_MAC_AG=2 HD_MAC_SPS=2 HD_MAC_PF=16
run ag4pf16 HD_MAC_AG=4 HD_MAC_PF=16
run ag4seppf16 HD_MAC_AG=4 HD_MAC_INLINE=0 HD_MAC_PF=16
