"""Development: where does a plain call's time go outside the CTAs' own timeline?  With a trace
build (L4_LIB=variants/libl4_trace.so): back-to-back per-call time, the CTA span (first entry ->
last done) of one call, and stream-ordered globaltimer stamps (1-thread kernels) around one call
and around 10 calls."""
import argparse
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2512_19179_b200 import l4


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c3")
    ap.add_argument("--uniform", type=int, nargs=2, default=None)
    args = ap.parse_args()
    spec = bench.WORKLOADS[args.workload]
    lens = spec["lens"]() if not args.uniform else np.full(args.uniform[0], args.uniform[1], dtype=np.int64)
    wl = bench.Workload(args.workload, lens, spec["shape"])
    p = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads)
    ws = l4.alloc_workspace(p, wl.table.total_pages)
    st = torch.cuda.current_stream()
    sh = ctypes.c_void_p(st.cuda_stream)
    fn = lambda: l4.attention_call(p, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len, wl.table.total_pages,
                                   wl.out, wl.lse, ws)
    lib = l4.lib()
    l4.decode_plan(p, wl.kv_len, wl.indptr, wl.table.total_pages, ws)  # header (num_ctas) for the trace read
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(30):
        fn()
    b.record()
    b.synchronize()
    per_call = a.elapsed_time(b) / 30 * 1e3
    # one call between stamps (the host enqueues everything first, then the GPU runs it)
    stamps = (ctypes.c_ulonglong * 64)()
    lib.l4_trace_clear()
    torch.cuda._sleep(2_000_000)  # keep the GPU busy while the host enqueues the sequence
    lib.l4_trace_stamp(0, sh)
    fn()
    lib.l4_trace_stamp(1, sh)
    for _ in range(10):
        fn()
    lib.l4_trace_stamp(2, sh)
    lib.l4_trace_stamp(3, sh)
    torch.cuda.synchronize()
    lib.l4_trace_read_stamps(stamps, 64)
    s = np.frombuffer(stamps, dtype=np.uint64)[:4].astype(np.float64)
    buf = (ctypes.c_ulonglong * (4096 * 16))()
    lib.l4_trace_read(buf, 4096 * 16)
    ncta = l4.plan_info(ws).num_ctas
    # the trace holds the LAST call's marks; stamps 1 -> 2 bracket the last 10 calls
    t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16)[:ncta, :10].astype(np.float64)
    entry, done = t[:, 0].min(), t[:, 5].max()
    print(f"{args.workload} {args.uniform or ''}: back-to-back {per_call:.1f} us/call; stamps: one call "
          f"{(s[1] - s[0]) / 1e3:.1f} us, ten calls {(s[2] - s[1]) / 1e4:.1f} us/call, empty stamp pair "
          f"{(s[3] - s[2]) / 1e3:.1f} us; last call: stamp1->first entry? CTA span {(done - entry) / 1e3:.1f} us, "
          f"last done -> stamp2 {(s[2] - done) / 1e3:.1f} us")


if __name__ == "__main__":
    main()
