#!/bin/bash
# Sweep of variant builds (LIBS="a b c": variants/libl4_<name>.so, "cur" = the in-tree libl4.so)
# over the headline and short-request workloads, plain / early-plan / early calls, two repeats.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-sweep}
for rep in 1 2; do
for W in "--workload c3" "--workload c4" "--workload c2" "--workload c2 --uniform 1024 64" "--workload c4 --uniform 1024 64" "--workload c2 --uniform 1024 200" ${EXTRA_WL}; do
  for n in ${LIBS:-base cur}; do
    if [ "$n" = cur ]; then LIB=paper_2512_19179_b200/libl4.so; else LIB=variants/libl4_$n.so; fi
    L4_LIB=$LIB timeout 300 python scripts/microbench.py $W --quick >> gpurun_out/${T}.log 2>&1
  done
done
done
python - <<'PY' gpurun_out/${T}.log
import sys, re, collections
d = collections.defaultdict(list)
for line in open(sys.argv[1]):
    m = re.match(r"(\S+ (?:\[[^\]]*\])?)\s*(\S+): plain ([\d.]+) us .*early-plan ([\d.]+) us .*early ([\d.]+) us", line)
    if m:
        d[(m.group(1).strip(), m.group(2).split('/')[-1])].append(tuple(float(m.group(i)) for i in (3, 4, 5)))
for k, v in d.items():
    print(f"{k[0]:18s} {k[1]:22s} plain {min(x[0] for x in v):8.2f}  eplan {min(x[1] for x in v):8.2f}  early {min(x[2] for x in v):8.2f}")
PY
