# quad threshold 1 / 2 vs the current 4 on batches with 1-3 quad units per CTA
cd $GRAFT_REPO_ROOT
for WL in c2 c4; do
for W in "--uniform 256 200" "--uniform 300 200" "--uniform 200 400" "--uniform 160 800" "--uniform 512 200" "--uniform 1024 64"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_qm1.so variants/libl4_qm2.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py --workload $WL $W --quick 2>&1 | tail -1
  done
done
done
for W in "--workload c3" "--workload c3 --bin 0 1024" "--workload c3 --bin 1024 4096"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_qm1.so variants/libl4_qm2.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
