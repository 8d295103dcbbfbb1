#!/bin/bash
# quad threshold sweep (quads per CTA required): homogeneous short batches of medium size
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
for B in 384 512 768; do
  for v in paper_2512_19179_b200/libl4.so scripts/var_m3.so scripts/var_m2.so; do
    echo "== B=$B $v"; L4_LIB=$v SB_BATCH=$B SB_LENS=64,200,530 timeout 200 python scripts/shortbench.py 2>&1 | tail -3
  done
done
