# bisect of the small mixed-batch regressions over the session's kernel commits (random sweep)
cd $GRAFT_REPO_ROOT
for LIB in variants/libl4_base.so variants/libl4_b35b34a5.so variants/libl4_b18c0cc1.so variants/libl4_b758f144.so variants/libl4_b629a5d1.so variants/libl4_b3ce02c6.so variants/libl4_bd0a286a.so paper_2512_19179_b200/libl4.so; do
  echo "== $LIB"; L4_LIB=$LIB RS_N=20 timeout 900 python scripts/randsweep.py 2>&1 | grep -E "case  (1|2|5|9|12|13|15|18) " | awk '{print $2, $(NF-3)}' | tr '\n' ' '; echo
done
