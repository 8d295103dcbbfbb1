cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for W in "--workload c4" "--workload c2 --uniform 25 39454" "--workload c2 --uniform 12 84547" "--workload c3"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_ipc12.so variants/libl4_ipc16.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick >> gpurun_out/r10.log 2>&1
  done
done
done
cat gpurun_out/r10.log
