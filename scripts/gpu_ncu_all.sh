#!/bin/bash
# ncu evidence for every bench workload, summarised on the box (the captures themselves exceed
# gpurun's copy-back limit): launch lists, summaries and DRAM traffic to gpurun_out/prof_summ,
# plus the C3 capture.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out/prof_summ
TAG=${TAG:-r2d}
WLS=${WLS:-"c3 c4 c2 short64 short200 short530 short70b_64 short70b_200 stage0 stage1024 stage4096 stage16384 stage65536"}
TAG=$TAG WLS="$WLS" bash scripts/gpu_ncu_r2.sh
PROF_OUT=gpurun_out/prof_summ python scripts/summarize_profiles.py $TAG $WLS > /dev/null 2>&1
ls gpurun_out/prof_summ
for f in gpurun_out/prof_${TAG}_*.ncu-rep; do case "$f" in *_c3.ncu-rep|*_short64.ncu-rep) ;; *) rm -f "$f";; esac; done
rm -f gpurun_out/launches_${TAG}_*.log gpurun_out/prof_${TAG}_*.log
du -sh gpurun_out
