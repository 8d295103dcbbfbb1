#!/bin/bash
# A/B of the in-tree libl4.so against variants/libl4_base.so (the previous kernel), plain /
# early-plan / early-input calls, headline and short-request workloads; parity tests first.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-ab}
if [ -z "$SKIP_TESTS" ]; then
  timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x > gpurun_out/${T}_pytest.log 2>&1; tail -3 gpurun_out/${T}_pytest.log
fi
for rep in 1 2; do
for W in "--workload c3" "--workload c4" "--workload c2" "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200" "--workload c2 --uniform 1024 530" "--workload c4 --uniform 1024 64" "--workload c4 --uniform 1024 200" ${EXTRA_WL}; do
  for LIB in variants/libl4_base.so paper_2512_19179_b200/libl4.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick >> gpurun_out/${T}.log 2>&1
  done
done
done
cat gpurun_out/${T}.log
if [ -n "$TRACE" ]; then
for W in "--workload c2" "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200"; do
  L4_LIB=variants/libl4_trace.so timeout 300 python scripts/trace_fused.py $W --mode fused >> gpurun_out/${T}_trace.log 2>&1
done
fi
