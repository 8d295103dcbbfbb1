#!/bin/bash
# planner latency study: micro-benchmarks + one full ncu capture of plan_kernel at C2
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_pipeline_gpu.py -q -m gpu > gpurun_out/pytest_pipe.log 2>&1; tail -2 gpurun_out/pytest_pipe.log
for w in c2 c3 c4; do timeout 300 python scripts/microbench.py --workload $w; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:plan_kernel -s 5 -c 1 \
  -o gpurun_out/prof_plan_c2 -f python scripts/microbench.py --workload c2 > gpurun_out/prof_plan.log 2>&1
tail -1 gpurun_out/prof_plan.log
