#!/bin/bash
# A/B of the committed kernel (scripts/var_base.so) vs the working tree (libl4.so) on small and headline batches
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 600 python -m pytest tests/test_decode_gpu.py -q -x --timeout 300 2>&1 | tail -1
for rep in 1 2; do
for a in "--workload c3 --bin 0 1024" "--workload c3 --bin 4096 16384" "--fig2 200 10000 1" "--uniform 256 200" "--workload c2"; do
  for v in scripts/var_base.so paper_2512_19179_b200/libl4.so; do L4_LIB=$v timeout 300 python scripts/microbench.py $a --quick; done
done; done
