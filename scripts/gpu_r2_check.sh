#!/bin/bash
# Round-2 check: GPU tests, smoke, default bench line.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-r2a}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu_${T}.log 2>&1; tail -5 gpurun_out/pytest_gpu_${T}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${T}.log 2>&1; tail -1 gpurun_out/smoke_${T}.log
timeout 900 python bench.py > gpurun_out/bench_${T}.log 2>&1; tail -c 3000 gpurun_out/bench_${T}.log
