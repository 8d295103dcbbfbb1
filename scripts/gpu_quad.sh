#!/bin/bash
# quad-unit A/B: parity tests of the default build, then short-batch and headline timings per variant
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_decode_gpu.py tests/test_stress_gpu.py -x -q --timeout 300 > gpurun_out/q_tests.log 2>&1; tail -3 gpurun_out/q_tests.log
for v in ${SB_VARIANTS:-scripts/var_q0.so scripts/var_q5.so paper_2512_19179_b200/libl4.so scripts/var_q6t0.so scripts/var_q6t4.so}; do
  echo "== $v"; L4_LIB=$v SB_LENS=${SB_LENS:-64,128,200,256,320,530,1024} timeout 200 python scripts/shortbench.py 2>&1 | tail -8
  L4_LIB=$v SB_BATCH=256 SB_LENS=64,200,530 timeout 200 python scripts/shortbench.py 2>&1 | tail -3
done
VARIANTS=${AB_VARIANTS:-"scripts/var_q0.so paper_2512_19179_b200/libl4.so scripts/var_q6t4.so"} timeout 900 bash scripts/gpu_ab.sh 2>&1
