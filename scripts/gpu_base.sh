cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -x > gpurun_out/pytest_gpu_base.log 2>&1; tail -3 gpurun_out/pytest_gpu_base.log
for W in "--workload c2" "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200"; do
  L4_LIB=variants/libl4_trace.so timeout 300 python scripts/trace_fused.py $W --mode fused >> gpurun_out/trace_base.log 2>&1
done
SB_LENS=64,200,530 timeout 300 python scripts/shortbench.py > gpurun_out/short_base.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_base.log 2>&1; tail -1 gpurun_out/bench_base.log | head -c 3000
