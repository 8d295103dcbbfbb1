# all-split chunk rule restricted to large batches: the C3 same-request bins, C4, long stages
cd $GRAFT_REPO_ROOT
for W in "--workload c3 --bin 4096 16384" "--workload c3 --bin 16384 65536" "--workload c3 --bin 65536 200000" "--workload c4" "--workload c2 --uniform 25 39454" "--workload c3"; do
  timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
done
