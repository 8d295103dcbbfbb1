cd $GRAFT_REPO_ROOT
for W in "--workload c3" "--workload c2" "--workload c4" "--workload c2 --uniform 1024 64"; do
  L4_LIB=variants/libl4_trace.so timeout 300 python scripts/gap_probe.py $W 2>&1 | tail -1
done
