#!/bin/bash
# Verify the proxy-fence fix: flake rates with the fixed debug build (per-call checksums) and the
# product build (bitwise repeats), plus forensics of the old build's wrong V slices.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
T=${TAG:-fixverify}
run() { echo "== $*" >> gpurun_out/${T}.log; timeout 1500 "$@" >> gpurun_out/${T}.log 2>&1; tail -1 gpurun_out/${T}.log; }
L4_LIB=variants/libl4_cks_nofence.so ITERS=3000 WANT=6 run python scripts/flake_forensic.py
L4_LIB=variants/libl4_cks.so run python scripts/flake_split.py --wl c4 --iters 3000 --cks --mode early
L4_LIB=variants/libl4_cks.so run python scripts/flake_split.py --wl c4 --iters 1500 --cks --mode plain
run python scripts/flake_split.py --wl c4 --iters 1500 --mode both
run python scripts/flake_split.py --wl c4 --iters 500 --poison --mode both
run python scripts/flake_split.py --wl c3 --iters 500 --mode both
