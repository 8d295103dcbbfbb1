# pipeline line at N = 1: host enqueue time per step vs device time per step
cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --pipeline --steps 30 --warmup 5 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())
for k,v in d['pipeline'].items(): print(k, round(v['kv_gbs']), 'elapsed/step', round(v['elapsed_ms']/30,3), 'busy/step', round(v['sum_busy_ms']/30,3), 'host/step', round(v['host_ms_per_step_max'],3))"
