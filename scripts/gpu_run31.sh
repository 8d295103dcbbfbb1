# chunk-search scratch aliased onto the bin counts (plan scratch back to its old size) vs HEAD
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x -k "c4 or long_stage or plan or fast_path" 2>&1 | tail -1
for rep in 1 2; do
for LIB in variants/libl4_prev.so paper_2512_19179_b200/libl4.so variants/libl4_base.so; do
  echo "== $LIB"; L4_LIB=$LIB RS_N=20 timeout 900 python scripts/randsweep.py 2>&1 | awk '{print $2, $(NF-3)}' | tr '\n' ' '; echo
  for W in "--workload c3" "--workload c4"; do L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1 | sed 's/early-plan.*//'; done
done
done
