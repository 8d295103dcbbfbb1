"""Development: plain-call device time of the final kernel vs a baseline build over seeded random
batch compositions (regression guard for the planner / quad heuristics).  L4_LIB selects the
library; run once per library and compare the printed lines."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import synth
from paper_2512_19179_b200 import l4


def timeit(fn, iters=30, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / iters * 1e3


def main():
    rng = np.random.default_rng(7)
    for case in range(int(os.environ.get("RS_N", "16"))):
        B = int(rng.choice([32, 64, 128, 256, 512, 768, 1024]))
        med = float(rng.choice([100, 300, 1000, 3000, 10000, 30000]))
        sig = float(rng.choice([0.3, 1.0, 1.5]))
        lens = np.clip(np.round(np.exp(rng.normal(np.log(med), sig, size=B))), 1, 131072).astype(np.int64)
        while lens.sum() * 4096 > 6e9:  # keep the pools within a few GB
            lens = np.maximum(1, lens // 2)
        shape = synth.SHAPE_LLAMA3_70B if rng.random() < 0.3 else synth.SHAPE_LLAMA3_8B
        wl = bench.Workload("rand", lens, shape)
        p = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads)
        ws = l4.alloc_workspace(p, wl.table.total_pages)
        fn = lambda: l4.attention_call(p, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len, wl.table.total_pages,
                                       wl.out, wl.lse, ws)
        t = timeit(fn)
        print(f"case {case:2d} {shape.name} B={B} med={med:.0f} sig={sig} sumL={int(lens.sum())}: {t:9.2f} us "
              f"{wl.bytes_kv / (t * 1e-6) / 1e9:7.0f} GB/s", flush=True)
        del wl, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
