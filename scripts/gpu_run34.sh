# is the residual mixed-batch cost the planner rewrite? final kernel with the start-of-session planner
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for LIB in variants/libl4_base.so variants/libl4_oldplan.so paper_2512_19179_b200/libl4.so; do
  echo "== $LIB"; L4_LIB=$LIB RS_N=20 timeout 900 python scripts/randsweep.py 2>&1 | awk '{print $2, $(NF-3)}' | tr '\n' ' '; echo
  for W in "--workload c3" "--workload c2"; do L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick 2>&1 | tail -1 | sed 's/early-plan.*//'; done
done
done
