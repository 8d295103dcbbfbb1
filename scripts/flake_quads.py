"""Development: bitwise repeat check of quad-unit launches in the few-quads-per-CTA regime
(B = 256 x ~200 tokens, G = 4 and 8), plain and early-input calls."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import synth
from paper_2512_19179_b200 import l4

N = int(os.environ.get("FN", "1000"))
for shape in (synth.SHAPE_LLAMA3_8B, synth.SHAPE_LLAMA3_70B):
    lens = np.random.default_rng(9).integers(150, 209, size=256)
    wl = bench.Workload("q", lens, shape)
    fails = 0
    for flags in (0, l4.L4_DECODE_EARLY_INPUTS):
        p = l4.make_params(256, shape.num_q_heads, shape.num_kv_heads, flags=flags)
        ws = l4.alloc_workspace(p, wl.table.total_pages)
        call = lambda o, s: l4.attention_call(p, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len,
                                              wl.table.total_pages, o, s, ws)
        ref_o, ref_l = torch.empty_like(wl.out), torch.empty_like(wl.lse)
        call(ref_o, ref_l)
        o, s = torch.empty_like(wl.out), torch.empty_like(wl.lse)
        for it in range(N):
            call(o, s)
            if it % 50 == 49:
                torch.cuda.synchronize()
                if not (torch.equal(o, ref_o) and torch.equal(s, ref_l)):
                    fails += 1
        torch.cuda.synchronize()
    print(f"{shape.name} B=256 x ~200: {2 * N} calls, {fails} mismatching checks", flush=True)
