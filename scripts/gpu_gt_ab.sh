#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
L4_LIB=variants/libl4_gt30_4.so timeout 1200 python -m pytest tests/test_decode_gpu.py -q --timeout 300 -x \
  -k "full_size_c3 or full_size_c4 or repeat or random_shapes or split or fused or two_level or longest" > gpurun_out/pytest_gt.log 2>&1
tail -2 gpurun_out/pytest_gt.log
TAG=gt_ab LIBS="paper_2512_19179_b200/libl4.so variants/libl4_gt20_2.so variants/libl4_gt20_4.so variants/libl4_gt30_4.so variants/libl4_gt40_4.so" TRACE_WLS="" \
  WLS="--workload%c4 --workload%c3 --workload%c2 --workload%c2%--uniform%25%39454 --workload%c2%--uniform%12%84547 --workload%c2%--uniform%183%5431 --workload%c2%--uniform%1024%200" \
  bash scripts/gpu_ab_cur.sh
