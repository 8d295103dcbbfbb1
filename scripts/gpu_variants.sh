#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for v in variants/*.so; do
  for w in c2 c3 c4; do echo "== $v $w"; L4_LIB=$PWD/$v timeout 300 python scripts/microbench.py --workload $w 2>&1 | tail -2; done
done
