# MAC TMA pipeline: parity tests, then A/B of the default step (TMA MAC vs the LDG kernel)
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2b_smoke.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_hardening.py tests/test_gpu_parity.py tests/test_gpu_batch.py tests/test_gpu_flat.py -m gpu -q -x > gpurun_out/r2b_pytest.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_default.log 2>&1
HD_MAC_VARIANT=c timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2b_classic.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --batch 4 > gpurun_out/r2b_batch4.log 2>&1
tail -n 3 gpurun_out/r2b_smoke.log gpurun_out/r2b_pytest.log
for f in gpurun_out/r2b_default.log gpurun_out/r2b_classic.log gpurun_out/r2b_batch4.log; do python - "$f" <<'PY'
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d.get('phase_ms_serial'), d['roofline']['frac'], d['query_roofline']['frac'])
PY
done
