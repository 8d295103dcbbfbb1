# forced-chunk sweep on uniform long stages: does a full last round (items = k x 296) shorten the tail?
cd $GRAFT_REPO_ROOT
for C in 0 60 67 80 97 110 124 130 139 146 155 165 178 190 208 230; do
  echo -n "25x39454 C=$C: "; timeout 300 python scripts/microbench.py --workload c2 --uniform 25 39454 --quick --chunk $C 2>&1 | tail -1 | sed 's/.*plain/plain/'
done
for C in 0 110 126 140 150 160 176 190 209 220 240 264 294 330; do
  echo -n "12x84547 C=$C: "; timeout 300 python scripts/microbench.py --workload c2 --uniform 12 84547 --quick --chunk $C 2>&1 | tail -1 | sed 's/.*plain/plain/'
done
