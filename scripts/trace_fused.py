"""Development timeline probe: run a trace build (L4_LIB=<variant .so built with -DL4_TRACE>)
and print, over CTAs, when each phase of decode_kernel happened (us from the earliest start):
0 entry, 1 after griddepcontrol.wait, 2 plan ready, 3 first TMA issued, 4 first page landed
(consumer warp 0), 5 CTA done; inside the planner: 6 loads + reduction, 7 chunk/count,
8 rank pass 1, 9 rank pass 2 (then offsets until 2)."""
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
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--mode", default="fused", choices=["fused", "run", "early"])
    ap.add_argument("--bin", type=int, nargs=2, default=None, help="only the workload's requests in [lo, hi)")
    ap.add_argument("--fig2", type=int, nargs=3, default=None, help="short long n_long: Fig. 2 batch of 512")
    ap.add_argument("--uniform", type=int, nargs=2, default=None, help="batch length: homogeneous batch")
    args = ap.parse_args()
    spec = bench.WORKLOADS[args.workload]
    lens = spec["lens"]()
    if args.bin:
        lens = lens[(lens >= args.bin[0]) & (lens < args.bin[1])]
    if args.fig2:
        import synth
        lens = synth.lengths_fig2(512, args.fig2[2], args.fig2[0], args.fig2[1])
    if args.uniform:
        lens = np.full(args.uniform[0], args.uniform[1], dtype=np.int64)
    wl = bench.Workload(args.workload, lens, spec["shape"])
    flags = l4.L4_DECODE_EARLY_INPUTS if args.mode == "early" else 0
    p = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads, flags=flags)
    ws = l4.alloc_workspace(p, wl.table.total_pages)
    l4.decode_plan(p, wl.kv_len, wl.indptr, wl.table.total_pages, ws)
    if args.mode in ("fused", "early"):
        fn = lambda: l4.attention_call(p, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len, wl.table.total_pages,
                                       wl.out, wl.lse, ws)
    else:
        fn = lambda: l4.decode_run(p, wl.q, wl.k, wl.v, wl.indices, wl.out, wl.lse, ws)
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    b.synchronize()
    ncta = l4.plan_info(ws).num_ctas
    l4.lib().l4_trace_clear()
    fn()
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (4096 * 16))()
    l4.lib().l4_trace_read(buf, 4096 * 16)
    t = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16)[:ncta, :10].astype(np.float64)
    t0 = t[:, 0].min()
    rel = (t - t0) / 1e3
    bytes_kv = wl.bytes_kv
    print(f"{args.workload} {args.bin} {args.mode}: {bytes_kv / 1e6:.0f} MB KV, event {a.elapsed_time(b) * 1e3:.1f} us, {ncta} CTAs")
    acc = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16)[:ncta, 12:16].astype(np.float64)
    acc2 = np.frombuffer(buf, dtype=np.uint64).reshape(4096, 16)[:ncta, 10:12].astype(np.float64)
    span = (t[:, 5] - t[:, 0]) / 1e3
    print(f"  per CTA (us, median over CTAs): busy {np.median(span):.1f}; consumer warp0 waiting for data "
          f"{np.median(acc[:, 0]) / 1e3:.1f}; item epilogues {np.median(acc[:, 1]) / 1e3:.1f}; producer waiting "
          f"for ring slots {np.median(acc[:, 2]) / 1e3:.1f}; items {np.median(acc[:, 3]):.0f} "
          f"(min {acc[:, 3].min():.0f}, max {acc[:, 3].max():.0f}); consumer warp0 waiting for the next item "
          f"(Q) {np.median(acc2[:, 0]) / 1e3:.1f}; warp0 page compute {np.median(acc2[:, 1]) / 1e3:.1f}")
    if hasattr(l4.lib(), "l4_trace_read_last"):
        lb = (ctypes.c_ulonglong * (4096 * 4))()
        l4.lib().l4_trace_read_last(lb, 4096 * 4)
        last = np.frombuffer(lb, dtype=np.uint64).reshape(4096, 4)[:ncta].astype(np.float64)
        ok = last[:, 0] > 0
        if not ok.any():
            ok = None
    if hasattr(l4.lib(), "l4_trace_read_last") and ok is not None:
        st = (last[ok, 0] - t0) / 1e3
        done = rel[ok, 5]
        print(f"  last CTA-wide item per CTA: start p10/p50/p90 {np.percentile(st, 10):.1f}/{np.median(st):.1f}/"
              f"{np.percentile(st, 90):.1f} us, pages p50 {np.median(last[ok, 1]):.0f} max {last[ok, 1].max():.0f}, "
              f"split {int((last[ok, 2] > 1).sum())}/{int(ok.sum())}; the 10 latest-finishing CTAs (done us, last "
              f"start us, pages, splits):")
        order = np.argsort(-done)[:10]
        print("   ", [(round(float(done[i]), 1), round(float(st[i]), 1), int(last[ok][i, 1]), int(last[ok][i, 2]))
                      for i in order])
    for k, name in enumerate(["entry", "pdl_wait", "plan", "tma0", "land0", "done", "p_load", "p_count", "p_pass1", "p_pass2"]):
        c = rel[:, k]
        c = c[(c > -1e6) & (c < 1e7)]  # marks a CTA never reached hold stale values
        if c.size == 0:
            continue
        print(f"  {name:9s} min {c.min():8.2f}  p50 {np.median(c):8.2f}  p90 {np.percentile(c, 90):8.2f}  max {c.max():8.2f}")


if __name__ == "__main__":
    main()
