# last-round fill chunk choice for large all-split batches (prev = fixed 12 items per CTA)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x > gpurun_out/r22_pytest.log 2>&1; tail -2 gpurun_out/r22_pytest.log
for rep in 1 2; do
for W in "--workload c4" "--workload c2 --uniform 25 39454" "--workload c2 --uniform 12 84547" "--workload c2 --uniform 64 16384" "--workload c2 --uniform 8 131072" "--workload c3"; do
  for LIB in variants/libl4_prev.so paper_2512_19179_b200/libl4.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
done
