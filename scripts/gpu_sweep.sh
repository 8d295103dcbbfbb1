#!/bin/bash
# development sweep over build variants (scripts/var_*.so) with microbench --quick
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in ${VARIANTS:-scripts/var_*.so}; do
  for w in c2 c3 c4; do L4_LIB=$v timeout 300 python scripts/microbench.py --workload $w --quick; done
  for b in "0 1024" "4096 16384" "16384 65536" "65536 1000000"; do L4_LIB=$v timeout 300 python scripts/microbench.py --workload c3 --bin $b --quick; done
done
