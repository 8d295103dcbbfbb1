# quad admission rule q_pages / 10 units per CTA (cur) vs min(4, q_pages / 4) (prev)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x > gpurun_out/r28_pytest.log 2>&1; tail -2 gpurun_out/r28_pytest.log
for WL in c2 c4; do
for W in "--uniform 256 200" "--uniform 300 200" "--uniform 200 400" "--uniform 400 400" "--uniform 160 800" "--uniform 512 200" "--uniform 1024 64" "--uniform 1024 200" "--uniform 1024 530"; do
  for LIB in variants/libl4_prev.so paper_2512_19179_b200/libl4.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py --workload $WL $W --quick 2>&1 | tail -1
  done
done
done
for W in "--workload c3" "--workload c2" "--workload c3 --bin 0 1024" "--workload c3 --bin 1024 4096" "--workload c2 --fig2 200 10000 8"; do
  for LIB in variants/libl4_prev.so paper_2512_19179_b200/libl4.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
