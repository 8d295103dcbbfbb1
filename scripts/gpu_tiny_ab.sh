#!/bin/bash
# tiny-item quads: committed kernel (scripts/var_base.so) vs working tree on small short batches
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_stress_gpu.py -q -x --timeout 600 2>&1 | tail -1
for B in 128 256 384 512; do
  for v in scripts/var_base.so paper_2512_19179_b200/libl4.so; do
    echo "== B=$B $v"; L4_LIB=$v SB_BATCH=$B SB_LENS=16,64,100 timeout 200 python scripts/shortbench.py 2>&1 | tail -3
  done
done
for a in "--workload c3 --bin 0 1024" "--fig2 200 10000 1" "--workload c3"; do
  for v in scripts/var_base.so paper_2512_19179_b200/libl4.so; do L4_LIB=$v timeout 300 python scripts/microbench.py $a --quick; done
done
