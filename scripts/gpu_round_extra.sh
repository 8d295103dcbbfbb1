#!/bin/bash
# round evidence, second half: the pipeline line at N = 1 and the N-rank harness on one GPU
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1d}
timeout 600 python bench.py --pipeline --steps 30 --warmup 5 > gpurun_out/bench_pipeline_${TAG}.log 2>&1; tail -1 gpurun_out/bench_pipeline_${TAG}.log | cut -c1-600
TRANSPORTS=ipc NS="2 4" timeout 1200 bash scripts/gpu_multirank.sh
