#!/bin/bash
# Split nondeterminism: per-item data checksums (debug variant) + flake rates.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-flake2}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 900 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
L4_LIB=variants/libl4_cks.so run python scripts/flake_split.py --wl c4 --iters 300 --cks --mode plain
L4_LIB=variants/libl4_cks.so run python scripts/flake_split.py --wl c4 --iters 200 --cks --mode early
