#!/bin/bash
# quick GPU iteration: parity tests + micro-benchmarks
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --timeout 180 -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
for w in ${WLS:-c2 c3 c4}; do timeout 300 python scripts/microbench.py --workload $w; done
