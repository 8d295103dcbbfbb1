# quad threshold (quads per CTA) between 2 and 4 on mid-size short batches
cd $GRAFT_REPO_ROOT
for W in "--uniform 300 200" "--uniform 400 200" "--uniform 450 100" "--uniform 400 400" "--uniform 600 64" "--uniform 300 100" "--uniform 700 300"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_qm2.so variants/libl4_qm3.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py --workload c2 $W --quick 2>&1 | tail -1
  done
done
for W in "--uniform 300 200" "--uniform 400 200"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_qm2.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py --workload c4 $W --quick 2>&1 | tail -1
  done
done
