#!/bin/bash
# ncu evidence of the quad-unit path: one launch on a B = 1024 batch of 200-token requests
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1d}
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:decode_kernel<.*bool.1>' -s 6 -c 1 -o gpurun_out/prof_${TAG}_short200 -f \
  python scripts/microbench.py --uniform 1024 200 --quick > gpurun_out/prof_${TAG}_short200.log 2>&1
tail -1 gpurun_out/prof_${TAG}_short200.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${TAG}_short200.csv python scripts/microbench.py --uniform 1024 200 --quick \
  > /dev/null 2>&1
