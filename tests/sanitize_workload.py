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
