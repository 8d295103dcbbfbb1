cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x > gpurun_out/r3_pytest.log 2>&1; tail -3 gpurun_out/r3_pytest.log
TAG=sw3 LIBS="base cur" EXTRA_WL="--workload c2 --uniform 256 200" bash scripts/gpu_variants_sweep.sh
for W in "--workload c3" "--workload c2 --uniform 1024 64"; do
  L4_LIB=variants/libl4_trace.so timeout 300 python scripts/trace_fused.py $W --mode fused >> gpurun_out/tr3.log 2>&1
done
grep -v "^ *\[" gpurun_out/tr3.log | grep -v "last CTA"
