"""Development: locate the (page, kv head) slices whose K / V data a call consumed differently from a
reference call (debug variant built with -DL4_DEBUG_PAGE), with where they were consumed."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2512_19179_b200 import l4

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=200)
ap.add_argument("--calls", type=int, default=3)
ap.add_argument("--early", type=int, default=1)
args = ap.parse_args()
shape, lens = synth.SHAPE_LLAMA3_70B, synth.lengths_c4(0)
table = synth.make_page_table(lens, seed=0, spare_pages=64)
g = torch.Generator(device="cuda").manual_seed(0)
B = table.batch
q = torch.randn(B, shape.num_q_heads, 128, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
ip, ix, kl = (torch.from_numpy(x).cuda() for x in (table.indptr, table.indices, table.kv_len))
N = table.num_pages * shape.num_kv_heads
owner = {}
for b in range(B):
    for j, p in enumerate(table.indices[table.indptr[b]:table.indptr[b + 1]]):
        owner[int(p)] = (b, j)


def read():
    pk = (ctypes.c_uint32 * N)()
    pv = (ctypes.c_uint32 * N)()
    meta = (ctypes.c_uint32 * (4 * N))()
    torch.cuda.synchronize()
    assert l4.lib().l4_debug_pages(pk, pv, meta, N) == 0
    return (np.frombuffer(pk, dtype=np.uint32).copy(), np.frombuffer(pv, dtype=np.uint32).copy(),
            np.frombuffer(meta, dtype=np.uint32).reshape(-1, 4).copy())


p0 = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads)
out, lse = l4.decode_attention(q, k, v, ip, ix, kl)
rk, rv, rm = read()
bad_total = 0
for it in range(args.iters):
    params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads, flags=l4.L4_DECODE_EARLY_INPUTS if args.early else 0)
    ws = l4.alloc_workspace(params, table.total_pages)
    o2, l2 = torch.empty_like(out), torch.empty_like(lse)
    for c in range(args.calls):
        l4.attention_call(params, q, k, v, ip, ix, kl, table.total_pages, o2, l2, ws)
        ck, cv, cm = read()
        bad = np.nonzero((ck != rk) | (cv != rv))[0]
        if len(bad):
            bad_total += 1
            for key in bad[:6]:
                page, h = divmod(int(key), shape.num_kv_heads)
                m = cm[key]
                print(f"iter {it} call {c}: page {page} h {h} (req, page#) {owner.get(page)}: K {'ok' if ck[key] == rk[key] else 'BAD'} "
                      f"V {'ok' if cv[key] == rv[key] else 'BAD'}; cta {m[0]} q {m[1]} (stage {m[1] % 8}) j {m[2] & 0xffff} "
                      f"warp {(m[2] >> 16) & 15} item# {m[2] >> 20} item {m[3]}", flush=True)
            # neighbours in the same CTA's ring (same cta, q within +-10)
            cta = cm[bad[0]][0]
            qq = int(cm[bad[0]][1])
            sel = np.nonzero((cm[:, 0] == cta) & (np.abs(cm[:, 1].astype(np.int64) - qq) <= 9))[0]
            rows = sorted((int(cm[s][1]), int(s)) for s in sel)
            print("   ring around: " + ", ".join(f"q{qv}:w{(cm[s][2] >> 16) & 15}:j{cm[s][2] & 0xffff}" for qv, s in rows), flush=True)
print(f"bad calls {bad_total} over {args.iters} iters x {args.calls} calls")
