#!/bin/bash
# ncu evidence: launch list of one bench command + one full capture of the dominant kernel.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
WL=${WL:-c2}
TAG=${TAG:-r1}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_${WL}.csv python bench.py --workload $WL --steps 3 --warmup 3 --no-extra --no-cpu \
  > gpurun_out/launches_${TAG}_${WL}.log 2>&1
tail -2 gpurun_out/launches_${TAG}_${WL}.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 4 -c 1 \
  -o gpurun_out/prof_${TAG}_${WL} -f python bench.py --workload $WL --steps 2 --warmup 3 --no-extra --no-cpu \
  > gpurun_out/prof_${TAG}_${WL}.log 2>&1
tail -3 gpurun_out/prof_${TAG}_${WL}.log
