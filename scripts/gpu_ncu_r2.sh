#!/bin/bash
# ncu evidence for the round: launch lists (gpu__time_duration.sum) of the bench command and one
# full capture of a steady-state decode_kernel launch per workload.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r2a}
for WL in ${WLS:-c3 c4 c2 short64 short200}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${WL}.csv python bench.py --workload $WL --steps 3 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/launches_${TAG}_${WL}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:decode_kernel<.*bool.1>' -s 6 -c 1 \
    -o gpurun_out/prof_${TAG}_${WL} -f python bench.py --workload $WL --steps 2 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/prof_${TAG}_${WL}.log 2>&1
  tail -1 gpurun_out/prof_${TAG}_${WL}.log | cut -c1-200
done
