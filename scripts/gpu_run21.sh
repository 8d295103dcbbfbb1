# forced-chunk sweep on C4 (items per CTA vs the fill of the last round)
cd $GRAFT_REPO_ROOT
for C in 0 300 320 340 360 385 400 420 440 460 480 500 520 550 576; do
  echo -n "c4 C=$C: "; timeout 300 python scripts/microbench.py --workload c4 --quick --chunk $C 2>&1 | tail -1 | sed 's/.*plain/plain/'
done
