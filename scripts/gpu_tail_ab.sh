#!/bin/bash
# Guided-tail variants vs the default build: plain / early-plan / early single-launch calls.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-tail_ab}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 600 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
for rep in 1 2; do
for V in ${VARIANTS:-default tail20_4 tail10_4 tail20_2 tail30_4 tail20_8}; do
  LIB=variants/libl4_$V.so; [ "$V" = default ] && LIB=paper_2512_19179_b200/libl4.so
  for W in "--workload c3" "--workload c4" "--workload c2" "--workload c2 --uniform 525 1890" \
           "--workload c2 --uniform 25 39454" "--workload c2 --uniform 1024 200" "--workload c2 --uniform 1024 64"; do
    L4_LIB=$LIB run python scripts/microbench.py $W --quick
  done
done
done
