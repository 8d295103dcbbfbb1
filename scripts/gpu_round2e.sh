#!/bin/bash
# Round-2 final evidence (kernel after the quad pacing / quad epilogue / planner fast path):
# GPU tests, smoke, default bench line, reference arm, read probe, ncu launch lists + summaries of
# every bench workload (+ the C3 and short64 captures), QoE re-fit, pipeline line at N = 1.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2e}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.log 2>&1; tail -c 600 gpurun_out/bench_${TAG}.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference_${TAG}.log 2>&1; tail -1 gpurun_out/bench_reference_${TAG}.log | cut -c1-300
[ -f scripts/readbw.so ] || bash scripts/build_readbw.sh > /dev/null 2>&1
python scripts/readbw.py > gpurun_out/readbw_${TAG}.json 2>&1
TAG=$TAG bash scripts/gpu_ncu_all.sh
timeout 900 python scripts/qoe_profile.py --tag $TAG > gpurun_out/qoe_${TAG}.log 2>&1; tail -2 gpurun_out/qoe_${TAG}.log
timeout 600 python bench.py --pipeline --steps 30 --warmup 5 > gpurun_out/bench_pipeline_${TAG}.log 2>&1; tail -c 400 gpurun_out/bench_pipeline_${TAG}.log
