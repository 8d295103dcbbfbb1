#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
L4_LIB=variants/libl4_ahead1.so timeout 1200 python -m pytest tests/test_decode_gpu.py -q --timeout 300 -x \
  -k "fused or quad or full_size_c3 or full_size_c4 or repeat or random_shapes or split" > gpurun_out/pytest_ahead1.log 2>&1
tail -2 gpurun_out/pytest_ahead1.log
for W in --workload%c3 --workload%c4; do
  for L in trace2 trace_a1; do
    L4_LIB=variants/libl4_$L.so timeout 300 python scripts/trace_fused.py ${W//%/ } --mode fused >> gpurun_out/ahead_trace.log 2>&1
  done
done
TAG=ahead_ab LIBS="paper_2512_19179_b200/libl4.so variants/libl4_ahead1.so" TRACE_WLS="" \
  WLS="--workload%c3 --workload%c4 --workload%c2 --workload%c2%--uniform%1024%64 --workload%c2%--uniform%1024%200 --workload%c2%--uniform%525%1890 --workload%c2%--uniform%25%39454" \
  bash scripts/gpu_ab_cur.sh
