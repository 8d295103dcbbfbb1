# re-sweeps on the final kernel: quad threshold (quads per CTA) and the mixed-batch chunk target
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for W in "--workload c3 --bin 0 1024" "--workload c2 --uniform 256 200" "--workload c2 --uniform 384 64" "--workload c2 --uniform 512 200" "--workload c2 --uniform 1024 64"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_qm2.so variants/libl4_qm3.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
for W in "--workload c3" "--workload c3 --bin 1024 4096" "--workload c2"; do
  for LIB in paper_2512_19179_b200/libl4.so variants/libl4_ipc6.so variants/libl4_ipc10.so; do
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1
  done
done
done
