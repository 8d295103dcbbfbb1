#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
cat > /tmp/sanit.py <<'PY'
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch, synth, bench
from paper_2512_19179_b200 import l4
lens = synth.lengths_c2()[: int(os.environ.get("NB", "250"))]
wl = bench.Workload("c2", lens, synth.SHAPE_LLAMA3_8B)
p = l4.make_params(len(wl.lens), 32, 8, chunk_pages=int(os.environ.get("CHUNK", "0")))
ws = l4.alloc_workspace(p, wl.table.total_pages)
l4.decode_plan(p, wl.kv_len, wl.indptr, wl.table.total_pages, ws)
info = l4.plan_info(ws)
print("items", info.num_items, "chunk", info.chunk_pages, "tail", info.tail_requests, info.tail_chunk_pages, flush=True)
l4.decode_run(p, wl.q, wl.k, wl.v, wl.indices, wl.out, wl.lse, ws)
torch.cuda.synchronize()
print("ok", float(wl.out.abs().max()))
PY
for cfg in "NB=250 CHUNK=-1" "NB=250 CHUNK=0" "NB=40 CHUNK=-1"; do
  echo "== $cfg"
  env $cfg timeout 300 compute-sanitizer --tool memcheck --print-limit 5 python /tmp/sanit.py 2>&1 | grep -v "^=========     Host Frame" | head -40
done
