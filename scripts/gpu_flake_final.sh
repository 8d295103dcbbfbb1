#!/bin/bash
# Final-kernel repeat checks (split-combine determinism after the early stage release and the
# chunk changes): every call's output (and, with --poison, NaN-filled split partials) compared
# bitwise with a reference call, C4 and C3, plain and early, plus the two-launch path.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-flake_final}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 1500 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
run python scripts/flake_split.py --wl c4 --iters 500 --poison --mode both
run python scripts/flake_split.py --wl c3 --iters 500 --poison --mode both
run python scripts/flake_split.py --wl c4 --iters 200 --poison --planrun
FN=400 run python scripts/flake_c4.py
