#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_pipeline_gpu.py tests/test_migrate_gpu.py -q --timeout 300 > gpurun_out/pytest_pipe.log 2>&1
tail -15 gpurun_out/pytest_pipe.log
timeout 600 python bench.py --pipeline --steps 20 --warmup 5 > gpurun_out/bench_pipe.log 2>&1
tail -3 gpurun_out/bench_pipe.log
