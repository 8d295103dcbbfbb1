cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x > gpurun_out/r11_pytest.log 2>&1; tail -3 gpurun_out/r11_pytest.log
TAG=sw11 LIBS="prev cur" EXTRA_WL="--workload c2 --uniform 25 39454 --workload c2 --uniform 12 84547" bash scripts/gpu_variants_sweep.sh
