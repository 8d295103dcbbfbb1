#!/bin/bash
# Per-CTA timelines (trace build) of plain single-launch calls: prologue, plan, first TMA, tail.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-trace}
for W in "--workload c2" "--workload c3" "--workload c4" "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200"; do
  L4_LIB=variants/libl4_trace.so timeout 300 python scripts/trace_fused.py $W --mode fused >> gpurun_out/${T}.log 2>&1
done
tail -60 gpurun_out/${T}.log
