# C2 variance check: the C2 main line twice, the extras' C2 entry in a full bench run, forced split chunk
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
timeout 300 python bench.py --workload c2 --steps 20 --warmup 5 --no-extra --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c2 main', d['ms_per_step'], d['value'])"
done
timeout 300 python scripts/microbench.py --workload c2 --quick | tail -1
timeout 300 python scripts/microbench.py --workload c2 --quick --chunk 32 | tail -1
timeout 300 python scripts/microbench.py --workload c2 --quick --chunk 43 | tail -1
timeout 900 python bench.py --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['roofline']['configs']; print('extras c2', c['c2']['ms'], c['c2']['kv_gbs'], 'c3', d['ms_per_step'])"
