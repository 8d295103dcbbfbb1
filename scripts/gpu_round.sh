#!/bin/bash
# Round evidence: default bench, launch lists and full ncu captures of the dominant kernel.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1}
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; tail -1 gpurun_out/bench_default_${TAG}.log
for WL in c2 c3 c4; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${WL}.csv python bench.py --workload $WL --steps 3 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/launches_${TAG}_${WL}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 6 -c 1 \
    -o gpurun_out/prof_${TAG}_${WL} -f python bench.py --workload $WL --steps 2 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/prof_${TAG}_${WL}.log 2>&1
  tail -1 gpurun_out/prof_${TAG}_${WL}.log
done
