B="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --no-size-curve --config C3 --packing flat --db encrypted --scenario membership"
for n in 23 128; do timeout 600 $B --n1 $n > gpurun_out/r5_paper_n$n.json 2>&1; python tools/bsum.py gpurun_out/r5_paper_n$n.json | cut -c1-100; done
timeout 600 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --no-size-curve --config C3 --packing flat_tbs --db encrypted --scenario membership --n1 23 > gpurun_out/r5_paper_tbs_n23.json 2>&1; python tools/bsum.py gpurun_out/r5_paper_tbs_n23.json | cut -c1-100
