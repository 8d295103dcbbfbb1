# A/B of the L2 input prefetch with the bench's rotating input copies (plain calls) + parity tests
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_decode_gpu.py -q --timeout 180 -x > gpurun_out/r17_pytest.log 2>&1; tail -2 gpurun_out/r17_pytest.log
for rep in 1 2; do
for WL in c3 c2 short64 short200 short70b_64 c4; do
  for LIB in variants/libl4_prev.so paper_2512_19179_b200/libl4.so; do
    L4_LIB=$LIB timeout 300 python bench.py --workload $WL --steps 20 --warmup 5 --no-extra --no-cpu 2>/dev/null | tail -1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$WL', '$LIB'.split('/')[-1], d['ms_per_step'], d['value'], d['roofline']['configs'].get('${WL}_cold'))"
  done
done
done
