# regression guard: seeded random batch compositions, final kernel vs the start-of-session build
cd $GRAFT_REPO_ROOT
for LIB in variants/libl4_base.so paper_2512_19179_b200/libl4.so; do
  echo "== $LIB"; L4_LIB=$LIB RS_N=20 timeout 900 python scripts/randsweep.py 2>&1 | tail -20
done
