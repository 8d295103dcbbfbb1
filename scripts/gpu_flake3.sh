#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-flake3}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 900 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
L4_LIB=variants/libl4_page.so run python scripts/flake_page.py --iters 150 --early 1
L4_LIB=variants/libl4_page.so run python scripts/flake_page.py --iters 100 --early 0
L4_LIB=variants/libl4_pfence.so run python scripts/flake_split.py --wl c4 --iters 300 --cks --mode early
