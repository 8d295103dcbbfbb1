#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for rep in 1 2; do
for a in "--workload c3 --bin 0 1024" "--fig2 200 10000 1" "--workload c2"; do
  for v in ${VARIANTS}; do L4_LIB=$v timeout 300 python scripts/microbench.py $a --quick; done
done
done
