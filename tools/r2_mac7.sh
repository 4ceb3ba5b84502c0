# 5-D single-box TMA MAC: variants + parity (C1/C2/C4 MAC paths)
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0"
run() { tag=$1; shift; env "$@" timeout 300 $B > gpurun_out/r2h_$tag.log 2>&1; python tools/bsum.py gpurun_out/r2h_$tag.log; }
run ag2s4 HD_MAC_AG=2 HD_MAC_SPS=4
run ag2s2 HD_MAC_AG=2 HD_MAC_SPS=2
run ag2s8 HD_MAC_AG=2 HD_MAC_SPS=8
run ag1s8 HD_MAC_AG=1 HD_MAC_SPS=8
run ag4s2 HD_MAC_AG=4 HD_MAC_SPS=2
run ag2s4dry HD_MAC_AG=2 HD_MAC_SPS=4 HD_MAC_TMA_DRY=1
run ag2s2dry HD_MAC_AG=2 HD_MAC_SPS=2 HD_MAC_TMA_DRY=1
timeout 300 python bench.py --no-cpu-baseline --steps 4 --warmup 2 --e2e-steps 0 --batch 4 > gpurun_out/r2h_b4.log 2>&1; python tools/bsum.py gpurun_out/r2h_b4.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_flat.py -m gpu -q -x -k "not c4" > gpurun_out/r2h_pytest.log 2>&1
tail -3 gpurun_out/r2h_pytest.log
