"""Small decode + migration workload run under compute-sanitizer by test_sanitizer_gpu.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2512_19179_b200 import l4

torch.cuda.init()
for G, Hkv, chunk in ((4, 2, 0), (8, 1, 2), (1, 3, -1)):
    lens = [0, 1, 15, 17, 300, 1000, 2500]
    shape = synth.AttnShape("s", G * Hkv, Hkv)
    t = synth.make_page_table(np.array(lens), seed=1, spare_pages=3)
    q, k, v = synth.make_qkv_cpu(shape, t, seed=1)
    out, lse = l4.decode_attention(q.cuda(), k.cuda(), v.cuda(), torch.from_numpy(t.indptr).cuda(),
                                   torch.from_numpy(t.indices).cuda(), torch.from_numpy(t.kv_len).cuda(),
                                   chunk_pages=chunk)
    torch.cuda.synchronize()
    assert torch.isfinite(out).all()
    # back-to-back single-launch calls with the early-input flag, then the two-launch path
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    ip, ix, kl = (torch.from_numpy(x).cuda() for x in (t.indptr, t.indices, t.kv_len))
    pe = l4.make_params(len(lens), G * Hkv, Hkv, chunk_pages=chunk, flags=l4.L4_DECODE_EARLY_INPUTS)
    ws = l4.alloc_workspace(pe, t.total_pages)
    o2, l2 = torch.empty_like(out), torch.empty_like(lse)
    for _ in range(3):
        l4.attention_call(pe, qd, kd, vd, ip, ix, kl, t.total_pages, o2, l2, ws)
    l4.decode_plan(pe, kl, ip, t.total_pages, ws)
    l4.decode_run(pe, qd, kd, vd, ix, o2, l2, ws)
    torch.cuda.synchronize()
    assert torch.equal(o2, out)
# quad units: 1024 short requests x 8 kv heads (>= 4 quads per CTA), a few long ones ahead;
# G = 4 (Q rows in the unit slot) and G = 8 (Q rows through the page ring)
for Hq in (32, 64):
    lens = np.random.default_rng(2).integers(1, 300, size=1024)
    lens[:3] = [5000, 0, 1]
    shape = synth.AttnShape("s", Hq, 8)
    t = synth.make_page_table(lens, seed=2, spare_pages=3)
    q, k, v = synth.make_qkv_cpu(shape, t, seed=2)
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    ip, ix, kl = (torch.from_numpy(x).cuda() for x in (t.indptr, t.indices, t.kv_len))
    pe = l4.make_params(len(lens), Hq, 8, flags=l4.L4_DECODE_EARLY_INPUTS)
    ws = l4.alloc_workspace(pe, t.total_pages)
    o1, l1 = torch.empty(len(lens), Hq, 128, device="cuda"), torch.empty(len(lens), Hq, device="cuda")
    o2, l2 = torch.empty_like(o1), torch.empty_like(l1)
    for _ in range(2):
        l4.attention_call(pe, qd, kd, vd, ip, ix, kl, t.total_pages, o1, l1, ws)
    l4.decode_plan(pe, kl, ip, t.total_pages, ws)
    l4.decode_run(pe, qd, kd, vd, ix, o2, l2, ws)
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.isfinite(o1).all()
# split-heavy, C4-like (Llama-3-70B shape: 64 q / 8 kv heads): long requests split up to 38 ways
# (two-level combine groups of 16), back-to-back early-input calls, NaN-poisoned split partials
lens = np.array([6000, 9000, 12000, 33])
shape = synth.AttnShape("s", 64, 8)
t = synth.make_page_table(lens, seed=3, spare_pages=3)
q, k, v = synth.make_qkv_cpu(shape, t, seed=3)
qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
ip, ix, kl = (torch.from_numpy(x).cuda() for x in (t.indptr, t.indices, t.kv_len))
ref, rl = l4.decode_attention(qd, kd, vd, ip, ix, kl, chunk_pages=20)
pe = l4.make_params(len(lens), 64, 8, chunk_pages=20, flags=l4.L4_DECODE_EARLY_INPUTS)
ws = l4.alloc_workspace(pe, t.total_pages)
l4.poison_partials(pe, ws)
o1, l1 = torch.empty_like(ref), torch.empty_like(rl)
for _ in range(3):
    l4.attention_call(pe, qd, kd, vd, ip, ix, kl, t.total_pages, o1, l1, ws)
torch.cuda.synchronize()
assert torch.equal(o1, ref) and torch.equal(l1, rl) and torch.isfinite(o1).all()
kk = torch.randn(2, 40, 2, 16, 128, device="cuda").to(torch.bfloat16)
vv = torch.randn_like(kk)
dk, dv = torch.zeros_like(kk), torch.zeros_like(vv)
pool = l4.PagePool(40)
l4.migrate(l4.kv_view(kk, vv, num_layers=2), [3, 9, 27], l4.kv_view(dk, dv, num_layers=2), pool)
st = torch.empty(3 * 2 * 2 * kk[0, 0].numel() * 2, dtype=torch.uint8, device="cuda")
l4.pack_pages(l4.kv_view(kk, vv, num_layers=2), [1, 2, 3], st)
l4.unpack_pages(l4.kv_view(dk, dv, num_layers=2), [4, 5, 6], st)
torch.cuda.synchronize()
print("SANITIZE_WORKLOAD_OK")
