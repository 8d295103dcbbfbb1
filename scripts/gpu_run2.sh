cd $GRAFT_REPO_ROOT
for W in "--workload c2" "--workload c3" "--workload c2 --uniform 1024 64" "--workload c4 --uniform 1024 64"; do
  L4_LIB=variants/libl4_trace.so timeout 300 python scripts/trace_fused.py $W --mode fused >> gpurun_out/tr2.log 2>&1
done
TAG=sw2 LIBS="base cur d8r4 d12r4" bash scripts/gpu_variants_sweep.sh
grep -v "^ *\[" gpurun_out/tr2.log | grep -v "last CTA" 
