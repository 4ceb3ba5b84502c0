mkdir -p gpurun_out/r4s
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 99 python -m pytest tests/test_gpu_parity.py -m gpu -q -x \
    -k "pipelined or streamed or toy_every_stage or level_reduced or ntt_bit_exact" > gpurun_out/r4s/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/r4s/sanitizer_$tool.log
done
