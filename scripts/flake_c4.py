"""Development: repeat the C4 early-vs-plain bitwise check in one process (intermittent mismatch hunt)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2512_19179_b200 import l4
shape = synth.SHAPE_LLAMA3_70B
lens = synth.lengths_c4(0)
table = synth.make_page_table(lens, seed=0, spare_pages=64)
g = torch.Generator(device="cuda").manual_seed(0)
B = table.batch
q = torch.randn(B, shape.num_q_heads, 128, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
ip, ix, kl = (torch.from_numpy(x).cuda() for x in (table.indptr, table.indices, table.kv_len))
out, lse = l4.decode_attention(q, k, v, ip, ix, kl)
fails = 0
N = int(os.environ.get("FN", "40"))
for it in range(N):
    params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads, flags=l4.L4_DECODE_EARLY_INPUTS if it % 2 else 0)
    ws = l4.alloc_workspace(params, table.total_pages)
    o2, l2 = torch.empty_like(out), torch.empty_like(lse)
    for _ in range(3):
        l4.attention_call(params, q, k, v, ip, ix, kl, table.total_pages, o2, l2, ws)
    torch.cuda.synchronize()
    if not (torch.equal(o2, out) and torch.equal(l2, lse)):
        fails += 1
        d = (o2 - out).abs()
        bad = (d.amax(dim=2) > 0).nonzero()
        print(f"iter {it} early={it % 2}: max diff {float(d.max()):.3e}, rows {bad[:6].tolist()} n={len(bad)}", flush=True)
print(os.environ.get("L4_LIB", "libl4.so"), f"fails {fails}/{N}")
