"""Development micro-benchmarks (device time via CUDA events): planner alone,
run alone, plan+run, for a named workload."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
from paper_2512_19179_b200 import l4


def timeit(fn, iters=50, warm=5):
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--chunk", type=int, default=0)
    ap.add_argument("--bin", type=int, nargs=2, default=None, help="only the workload's requests in [lo, hi)")
    ap.add_argument("--quick", action="store_true", help="fused / early only")
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
    p = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads, chunk_pages=args.chunk)
    ws = l4.alloc_workspace(p, wl.table.total_pages)
    plan = lambda: l4.decode_plan(p, wl.kv_len, wl.indptr, wl.table.total_pages, ws)
    run = lambda: l4.decode_run(p, wl.q, wl.k, wl.v, wl.indices, wl.out, wl.lse, ws)
    both = lambda: (plan(), run())
    fused = lambda: l4.attention_call(p, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len, wl.table.total_pages,
                                      wl.out, wl.lse, ws)
    pe = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads, chunk_pages=args.chunk,
                        flags=l4.L4_DECODE_EARLY_INPUTS)
    early = lambda: l4.attention_call(pe, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len, wl.table.total_pages,
                                      wl.out, wl.lse, ws)
    pp = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads, chunk_pages=args.chunk,
                        flags=getattr(l4, "L4_DECODE_EARLY_PLAN", 0))
    eplan = lambda: l4.attention_call(pp, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len, wl.table.total_pages,
                                      wl.out, wl.lse, ws)
    plan()
    if args.quick:
        t_fused, t_eplan, t_early = timeit(fused), timeit(eplan), timeit(early)
        gb = lambda t: wl.bytes_kv / (t * 1e-6) / 1e9
        print(f"{args.workload} {args.bin or args.fig2 or args.uniform or ''} {os.environ.get('L4_LIB', 'libl4.so')}: "
              f"plain {t_fused:.2f} us ({gb(t_fused):.0f} GB/s), early-plan {t_eplan:.2f} us ({gb(t_eplan):.0f}), "
              f"early {t_early:.2f} us ({gb(t_early):.0f})")
        return
    t_plan = timeit(plan)
    t_run = timeit(run)
    t_both = timeit(both)
    t_fused = timeit(fused)
    def timeit_ev(fn, iters=50, warm=5):  # an event recorded after every call
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(iters + 1)]
        evs[0].record()
        for i in range(iters):
            fn()
            evs[i + 1].record()
        evs[-1].synchronize()
        return evs[0].elapsed_time(evs[-1]) / iters * 1e3
    print(f"  per-call events: fused {timeit_ev(fused):.2f} us, early {timeit_ev(early):.2f} us")
    t_early = timeit(early)
    # device-only cost: the same calls captured in a CUDA graph (no host launch overhead)
    def graph_time(fn, reps=20):
        s = torch.cuda.Stream()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            fn()
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
        return timeit(g.replay, iters=10, warm=2) / reps
    try:
        g_plan, g_run, g_both, g_fused = graph_time(plan), graph_time(run), graph_time(both), graph_time(fused)
        g_early = graph_time(early)
        print(f"  graph: plan {g_plan:.2f} us, run {g_run:.2f} us, plan+run {g_both:.2f} us "
              f"({wl.bytes_kv / (g_both * 1e-6) / 1e9:.0f} GB/s), fused {g_fused:.2f} us "
              f"({wl.bytes_kv / (g_fused * 1e-6) / 1e9:.0f} GB/s), early {g_early:.2f} us "
              f"({wl.bytes_kv / (g_early * 1e-6) / 1e9:.0f} GB/s)")
    except Exception as e:  # noqa
        print("  graph capture failed:", e)
    info = l4.plan_info(ws)
    gbs = wl.bytes_kv / (t_both * 1e-6) / 1e9
    print(f"{args.workload}: plan {t_plan:.2f} us, run {t_run:.2f} us ({wl.bytes_kv / (t_run * 1e-6) / 1e9:.0f} GB/s), "
          f"plan+run {t_both:.2f} us ({gbs:.0f} GB/s), fused {t_fused:.2f} us "
          f"({wl.bytes_kv / (t_fused * 1e-6) / 1e9:.0f} GB/s), early {t_early:.2f} us "
          f"({wl.bytes_kv / (t_early * 1e-6) / 1e9:.0f} GB/s); items {info.num_items} chunk {info.chunk_pages}")


if __name__ == "__main__":
    main()
