#!/bin/bash
# repeat a GPU test selection to catch intermittent failures; keeps the log of the first failure
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
N=${N:-20}; SEL=${SEL:-"tests/test_c_abi.py tests/test_decode_gpu.py"}; K=${K:-}
fails=0
for i in $(seq 1 $N); do
  timeout 900 python -m pytest $SEL -q -x --timeout 600 ${K:+-k "$K"} > gpurun_out/rep_$i.log 2>&1
  rc=$?
  if [ $rc -ne 0 ]; then fails=$((fails+1)); cp gpurun_out/rep_$i.log gpurun_out/rep_fail_$fails.log; grep -n "^E " gpurun_out/rep_$i.log | head -12; fi
  rm -f gpurun_out/rep_$i.log
done
echo "runs=$N fails=$fails"
