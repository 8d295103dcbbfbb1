#!/bin/bash
# Proxy-fence placement: flake rates (debug checksum builds) and speed (plain builds).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-fence_ab}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 1200 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
L4_LIB=variants/libl4_rawfence.so run python scripts/flake_split.py --wl c4 --iters 1500 --cks --mode early
for rep in 1 2; do
for V in libl4.so variants/libl4_pfence_nocks.so variants/libl4_rawfence_nocks.so; do
  for W in "--workload c2" "--workload c3" "--workload c4" "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200"; do
    L4_LIB=$([ "$V" = libl4.so ] && echo paper_2512_19179_b200/libl4.so || echo $V) run python scripts/microbench.py $W --quick
  done
done
done
