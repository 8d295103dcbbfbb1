#!/bin/bash
# development iteration: decode parity tests, trace timelines, micro-benchmarks
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
timeout 600 python -m pytest tests/test_decode_gpu.py -q -x --timeout 300 2>&1 | tail -3
for w in ${TRACE_WLS:-c2}; do L4_LIB=scripts/trace.so python scripts/trace_fused.py --workload $w --mode fused; done
for w in ${WLS:-c2 c3 c4}; do timeout 300 python scripts/microbench.py --workload $w; done
