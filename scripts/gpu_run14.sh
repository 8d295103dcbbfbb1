cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/r14_pytest.log 2>&1; tail -3 gpurun_out/r14_pytest.log
timeout 900 python bench.py > gpurun_out/bench_r14.log 2>&1; tail -1 gpurun_out/bench_r14.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value']); print(json.dumps(d['summary']))"
