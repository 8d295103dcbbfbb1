#!/bin/bash
# Split-combine nondeterminism hunt (scripts/flake_split.py) on the base library and variants.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-flake}
ITERS=${ITERS:-100}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 900 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
run python scripts/flake_split.py --wl c4 --iters $ITERS
run python scripts/flake_split.py --wl c4 --iters $ITERS --poison
run python scripts/flake_split.py --wl c4 --iters $ITERS --planrun
for V in ${VARIANTS}; do
  L4_LIB=variants/$V.so run python scripts/flake_split.py --wl c4 --iters $ITERS
done
run python scripts/flake_split.py --wl c3 --iters $((ITERS/2))
