B="python bench.py --no-cpu-baseline --steps 20 --warmup 5 --e2e-steps 0 --no-size-curve --no-check"
for n1 in 256 64; do timeout 300 $B --n1 $n1 > gpurun_out/r3m_n$n1.log 2>&1; python tools/bsum.py gpurun_out/r3m_n$n1.log; done
timeout 300 $B --packing flat --n1 256 > gpurun_out/r3m_flat256.log 2>&1; python tools/bsum.py gpurun_out/r3m_flat256.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kip_giant -c 1 -o gpurun_out/r3m_kipg python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:kip_kernel -c 1 -o gpurun_out/r3m_kip python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 --no-size-curve --no-check > /dev/null 2>&1
ls gpurun_out/r3m*
