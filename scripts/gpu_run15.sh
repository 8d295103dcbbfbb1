# G = 8 quad Q rows: loaded by the consumers from global (cur) vs through the ring (qring); pacing
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x > gpurun_out/r15_pytest.log 2>&1; tail -3 gpurun_out/r15_pytest.log
for rep in 1 2; do
for W in "--workload c4 --uniform 1024 64" "--workload c4 --uniform 1024 200" "--workload c4 --uniform 1024 530" "--workload c4 --uniform 512 64" "--workload c4"; do
  for LIB in variants/libl4_qring.so paper_2512_19179_b200/libl4.so variants/libl4_qd16.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick >> gpurun_out/r15.log 2>&1
  done
done
done
cat gpurun_out/r15.log
