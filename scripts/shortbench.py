"""Development: single-launch decode time on homogeneous batches of short requests
(per-item overheads and the pages-per-consumer-warp quantisation of short items)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2512_19179_b200 import l4


def timeit(fn, iters=40, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / iters * 1e3  # us


def main():
    import synth
    shape = synth.SHAPE_LLAMA3_70B if os.environ.get("SB_SHAPE") == "70b" else bench.WORKLOADS["c2"]["shape"]
    B = int(os.environ.get("SB_BATCH", "1024"))
    lengths = [int(x) for x in os.environ.get("SB_LENS", "64,128,176,192,200,208,240,256,320,512,530,1024").split(",")]
    for L in lengths:
        wl = bench.Workload("c2", np.full(B, L, dtype=np.int64), shape)
        pe = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads, flags=l4.L4_DECODE_EARLY_INPUTS)
        ws = l4.alloc_workspace(pe, wl.table.total_pages)
        early = lambda: l4.attention_call(pe, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len,
                                          wl.table.total_pages, wl.out, wl.lse, ws)
        t = timeit(early)
        info = l4.plan_info(ws)
        print(f"L={L:5d} B={B} pages/req={(L + 15) // 16:3d}: {t:8.2f} us {wl.bytes_kv / (t * 1e-6) / 1e9:7.0f} GB/s "
              f"items {info.num_items} chunk {info.chunk_pages}", flush=True)
        del wl, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
