# planner loops back to tile-by-tile (cur: per-lane atomics; agg: match_any-aggregated) vs unrolled (prev) and the old planner
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x 2>&1 | tail -1
for rep in 1 2; do
for LIB in variants/libl4_prev.so variants/libl4_oldplan.so variants/libl4_agg.so paper_2512_19179_b200/libl4.so; do
  echo "== $LIB"; L4_LIB=$LIB RS_N=20 timeout 900 python scripts/randsweep.py 2>&1 | awk '{print $2, $(NF-3)}' | tr '\n' ' '; echo
  for W in "--workload c3" "--workload c2" "--workload c2 --uniform 1024 64" "--workload c4"; do L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1 | sed 's/early-plan.*//'; done
done
done
