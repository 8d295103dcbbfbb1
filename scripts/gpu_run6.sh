cd $GRAFT_REPO_ROOT
for rep in 1 2 3; do
for W in "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200"; do
  for LIB in variants/libl4_nullplan.so paper_2512_19179_b200/libl4.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick >> gpurun_out/r6.log 2>&1
  done
done
done
cat gpurun_out/r6.log
