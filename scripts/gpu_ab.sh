#!/bin/bash
# A/B of two builds (scripts/var_old.so vs scripts/var_new.so) on the headline and small workloads
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for a in "--workload c2" "--workload c3" "--workload c4" "--workload c3 --bin 0 1024" "--workload c3 --bin 16384 65536" "--fig2 200 10000 1" "--fig2 200 10000 32" "--uniform 1024 530"; do
  for v in ${VARIANTS:-scripts/var_old.so scripts/var_new.so}; do L4_LIB=$v timeout 300 python scripts/microbench.py $a --quick; done
done
