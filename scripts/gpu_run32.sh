# is the mixed-batch regression code layout? chunk search compiled out vs in
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for LIB in variants/libl4_base.so variants/libl4_nosearch.so paper_2512_19179_b200/libl4.so; do
  echo "== $LIB"; L4_LIB=$LIB RS_N=20 timeout 900 python scripts/randsweep.py 2>&1 | awk '{print $2, $(NF-3)}' | tr '\n' ' '; echo
  L4_LIB=$LIB timeout 300 python scripts/microbench.py --workload c3 --quick 2>&1 | tail -1 | sed 's/early-plan.*//'
done
done
