# no-compute skeleton A/B (variants/libl4_nocomp.so: -DL4_NO_COMPUTE)
cd $GRAFT_REPO_ROOT
for W in "--workload c3" "--workload c4" "--workload c2" "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_nocomp.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
