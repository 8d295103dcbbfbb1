cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/r4_pytest.log 2>&1; tail -3 gpurun_out/r4_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k 'regex:decode_kernel<.*bool.1>' -s 6 -c 1 \
    -o gpurun_out/prof_r4_short64 -f python bench.py --workload short64 --steps 2 --warmup 3 --no-extra --no-cpu \
    > gpurun_out/prof_r4_short64.log 2>&1
tail -2 gpurun_out/prof_r4_short64.log | cut -c1-300
ncu -i gpurun_out/prof_r4_short64.ncu-rep --page source --csv --print-source sass,cuda > gpurun_out/src_r4_short64.csv 2>&1 || ncu -i gpurun_out/prof_r4_short64.ncu-rep --page source --csv > gpurun_out/src_r4_short64.csv 2>&1
ls -la gpurun_out/
