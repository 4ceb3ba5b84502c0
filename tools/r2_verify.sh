# Round-2 verification on one B200: smoke, all GPU tests, sanitizers, bench lines, ncu evidence
set -x
mkdir -p gpurun_out/r2v
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2v/smoke.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2v/pytest_gpu.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
    -k "pipelined or streamed or toy_every_stage or level_reduced" > gpurun_out/r2v/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2v/sanitizer_rc.txt
done
timeout 600 python bench.py > gpurun_out/r2v/default.log 2>&1
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2v/ref.log 2>&1
timeout 600 python bench.py --packing flat --no-cpu-baseline > gpurun_out/r2v/flat.log 2>&1
timeout 600 python bench.py --batch 4 --no-cpu-baseline --steps 8 > gpurun_out/r2v/batch4.log 2>&1
timeout 900 python bench.py --config C3 --profile paper --no-cpu-baseline > gpurun_out/r2v/paper_C3.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/r2v/launches_default.csv python bench.py --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-check > gpurun_out/r2v/ncu_launches.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:mac_tma -c 1 --csv \
  --log-file gpurun_out/r2v/mac_traffic.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-check > gpurun_out/r2v/ncu_traffic.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mac_tma -c 1 -o gpurun_out/r2v/mac_tma_full \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-check > gpurun_out/r2v/ncu_full.log 2>&1
tail -n 2 gpurun_out/r2v/smoke.log gpurun_out/r2v/pytest_gpu.log; cat gpurun_out/r2v/sanitizer_rc.txt
python tools/bsum.py gpurun_out/r2v/default.log gpurun_out/r2v/flat.log gpurun_out/r2v/batch4.log gpurun_out/r2v/paper_C3.log
