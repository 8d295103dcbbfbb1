#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-flake4}
IT=${ITERS:-1500}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 1200 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
for V in cks pfence vearly allarrive cks pfence; do
  L4_LIB=variants/libl4_$V.so run python scripts/flake_split.py --wl c4 --iters $IT --cks --mode early
done
