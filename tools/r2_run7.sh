# the N > 1 bench path on one GPU (gloo, both ranks on cuda:0; test aid, not a bench number),
# the online-aggregated membership with the query rescaling, and the new compare test
export HD_BENCH_ONE_GPU=1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config C2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_n2_C2.log 2>&1; echo "n2 C2 rc=$?"; tail -c 1500 gpurun_out/r2m_n2_C2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2m_n2_C4.log 2>&1; echo "n2 C4 rc=$?"; tail -c 1500 gpurun_out/r2m_n2_C4.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --packing flat --scenario membership > gpurun_out/r2m_n2_mem.log 2>&1; echo "n2 mem rc=$?"; tail -c 800 gpurun_out/r2m_n2_mem.log
unset HD_BENCH_ONE_GPU
timeout 600 python bench.py --no-cpu-baseline --steps 10 --scenario membership --packing flat --db encrypted --online-aggregate > gpurun_out/r2m_aggr.log 2>&1; python tools/bsum.py gpurun_out/r2m_aggr.log
timeout 900 python -m pytest tests/test_gpu_compare.py -m gpu -q -x > gpurun_out/r2m_pytest_compare.log 2>&1; tail -3 gpurun_out/r2m_pytest_compare.log
