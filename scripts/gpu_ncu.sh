#!/bin/bash
# ncu only: launch lists + one full capture of the single-launch decode kernel per workload
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1b}
for WL in ${WLS:-c2 c3 c4}; do
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:decode_kernel<.*bool.1>' -s 4 -c 1 \
    -o gpurun_out/prof_${TAG}_${WL} -f python bench.py --workload $WL --steps 2 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/prof_${TAG}_${WL}.log 2>&1
  tail -1 gpurun_out/prof_${TAG}_${WL}.log | cut -c1-200
done
