# quad tail re-test: the last L4_QUAD_TAIL x W items of the quad suffix run CTA-wide
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for W in "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200" "--workload c2 --uniform 1024 530" "--workload c4 --uniform 1024 64" "--workload c2 --uniform 512 64"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_qt1.so variants/libl4_qt2.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
done
