# Round-end verification on one B200 (gpurun): smoke, every GPU test, the bench lines of
# every mode, the reference arm and a launch list of the default step.
set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/final_default.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_ref.log 2>&1
timeout 500 python bench.py --packing flat --no-cpu-baseline > gpurun_out/final_flat.log 2>&1
timeout 500 python bench.py --batch 2 --no-cpu-baseline > gpurun_out/final_batch2.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_default.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline > gpurun_out/final_ncu.log 2>&1
tail -n 2 gpurun_out/final_smoke.log gpurun_out/final_pytest_gpu.log
