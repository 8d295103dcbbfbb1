cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py tests/test_c_abi.py tests/test_pipeline_gpu.py -q --timeout 300 -x > gpurun_out/r16_pytest.log 2>&1; tail -3 gpurun_out/r16_pytest.log
for W in "--workload c4 --uniform 1024 64" "--workload c4 --uniform 1024 200" "--workload c4" "--workload c2 --uniform 1024 64" "--workload c3"; do
  for LIB in variants/libl4_qring.so paper_2512_19179_b200/libl4.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
