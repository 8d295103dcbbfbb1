# plan / run / plan+run / fused / early device times (materialised plan reuse across layers)
cd $GRAFT_REPO_ROOT
for W in "--workload c3" "--workload c2" "--workload c4" "--workload c2 --uniform 1024 64" "--workload c2 --uniform 1024 200"; do
  timeout 300 python scripts/microbench.py $W 2>&1 | tail -3
done
