# TMA MAC diagnosis: dry run (stream only), stage / AG variants, ncu --set full of the kernel
set -x
B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --e2e-steps 0"
summ() { python - "$1" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], round(d['value'],2), 'mac', round(d['phase_ms_serial']['mac'],3))
PY
}
timeout 300 $B > gpurun_out/r2c_default.log 2>&1; summ gpurun_out/r2c_default.log
HD_MAC_TMA_DRY=1 timeout 300 $B > gpurun_out/r2c_dry.log 2>&1; summ gpurun_out/r2c_dry.log
HD_MAC_AG=1 timeout 300 $B > gpurun_out/r2c_ag1.log 2>&1; summ gpurun_out/r2c_ag1.log
HD_MAC_STAGES=3 timeout 300 $B > gpurun_out/r2c_st3.log 2>&1; summ gpurun_out/r2c_st3.log
HD_MAC_TMA_DRY=1 HD_MAC_STAGES=3 timeout 300 $B > gpurun_out/r2c_dry3.log 2>&1; summ gpurun_out/r2c_dry3.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mac_tma -c 1 -o gpurun_out/r2c_mac_tma python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 > gpurun_out/r2c_ncu.log 2>&1
tail -3 gpurun_out/r2c_ncu.log
timeout 900 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_flat.py -m gpu -q -x > gpurun_out/r2c_pytest.log 2>&1
tail -3 gpurun_out/r2c_pytest.log
