#!/bin/bash
# A/B of the working tree's build against the last commit's (variants/libl4_head.so), + trace.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-ab_cur}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 600 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
# workloads: space-separated lists, '%' standing for a space inside one workload
for W in ${TRACE_WLS:---workload%c2 --workload%c2%--uniform%1024%64}; do
  L4_LIB=variants/libl4_trace2.so timeout 300 python scripts/trace_fused.py ${W//%/ } --mode fused >> gpurun_out/${T}_trace.log 2>&1
done
for rep in 1 2; do
for LIB in ${LIBS:-variants/libl4_head.so paper_2512_19179_b200/libl4.so}; do
  for W in ${WLS:---workload%c3 --workload%c2 --workload%c2%--uniform%1024%200 --workload%c2%--uniform%1024%64}; do
    L4_LIB=$LIB run python scripts/microbench.py ${W//%/ } --quick
  done
done
done
