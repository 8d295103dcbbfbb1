#!/bin/bash
# Round evidence: GPU tests, smoke, default bench, launch lists and full ncu captures of the
# dominant kernel (the single-launch decode_kernel<G, true>).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-r1b}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/pytest_gpu_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_gpu_${TAG}.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
timeout 900 python bench.py > gpurun_out/bench_default_${TAG}.log 2>&1; tail -1 gpurun_out/bench_default_${TAG}.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference_${TAG}.log 2>&1; tail -1 gpurun_out/bench_reference_${TAG}.log | cut -c1-300
python scripts/readbw.py > gpurun_out/readbw_${TAG}.json 2>&1
for WL in ${WLS:-c2 c3 c4}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${TAG}_${WL}.csv python bench.py --workload $WL --steps 3 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/launches_${TAG}_${WL}.log 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:decode_kernel<.*bool.1>' -s 4 -c 1 \
    -o gpurun_out/prof_${TAG}_${WL} -f python bench.py --workload $WL --steps 2 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/prof_${TAG}_${WL}.log 2>&1
  tail -1 gpurun_out/prof_${TAG}_${WL}.log | cut -c1-200
done
