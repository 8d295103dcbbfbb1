#!/usr/bin/env python3
"""bench.py — L4 hot path on B200: decode-attention KV GB/s (% of HBM peak).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4] [--impl l4|reference]

A step is one pass of the hot path over one synthetic batch: one
l4_decode_attention call = the length-binned work-list build (a1, done by every
CTA in shared memory) + the split-KV kernel with its fused LSE combine (a2+a3),
in ONE launch, i.e. one decode iteration of one layer.
`value` = algorithmic KV bytes per step / device time (GB/s), inputs resident
in HBM; `e2e` = the same metric through the public API with host buffers
(q, kv_len and the page table copied H2D, the output D2H, every step).
The KV working set (1-11 GB) exceeds the 126 MB L2, so no flush is needed.

N > 1 (torchrun): every rank runs its own instance (replicas of the same
workload, no data-path collective, "weak" scaling); time = max over ranks.

--impl reference: the FP64 CPU oracle (oracle/attention.py), as it stands, on
a bounded sample of the same workload — the reference arm for this tier.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOADS = {
    "c2": dict(desc="BASELINE configs[1]: Llama-3-8B attention (32q/8kv, d128), bf16, batch 250, uniform 1K contexts",
               shape=synth.SHAPE_LLAMA3_8B, lens=lambda: synth.lengths_c2()),
    "c3": dict(desc="BASELINE configs[2]: Llama-3-8B shape, batch 256, ShareGPT-like skewed 100..128K (seed 0), mixed batch",
               shape=synth.SHAPE_LLAMA3_8B, lens=lambda: synth.lengths_c3(0)),
    "c4": dict(desc="BASELINE configs[3]: Llama-3-70B attention (64q/8kv), long-context batch 32, 32K..128K (seed 0)",
               shape=synth.SHAPE_LLAMA3_70B, lens=lambda: synth.lengths_c4(0)),
}
METRIC = "decode-attn KV GB/s (% HBM peak), mixed vs binned; tokens/s at 1/2/4/8 GPUs"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_ceiling():
    """HBM read ceiling measured on this pool by the development probe (scripts/readbw.py:
    128-bit loads and TMA bulk reads of 1-4 GB, committed as profiles/readbw_r*.json), for
    context: the decode kernel only reads, the roofline peak stays MEASURED_PEAKS.json's copy."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "readbw_r*.json")))
    for f in reversed(files):
        try:
            d = json.load(open(f))
        except ValueError:
            continue
        vals = [v for k, v in d.items() if not k.startswith("copy") and isinstance(v, (int, float))]
        if vals:
            return float(max(vals)), os.path.relpath(f, ROOT)
    return None, None


def measured_traffic(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one decode_kernel launch from the
    committed ncu --set full capture (profiles/*_traffic.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    for f in reversed(files):
        d = json.load(open(f))
        if workload in d:
            return int(d[workload]["traffic"]), os.path.relpath(f, ROOT)
    return None, None


def kv_bytes(lens, shape) -> int:
    return int(4 * shape.num_kv_heads * shape.head_dim * int(np.sum(lens)))


def algo_bytes(lens, shape) -> int:
    """K+V once + q (bf16) + out (fp32) + page indices."""
    B = len(lens)
    pages = sum(synth.pages_for(x) for x in lens)
    return kv_bytes(lens, shape) + B * shape.num_q_heads * 128 * (2 + 4) + 4 * pages


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for n, flag in zip(names, parts[5:9]):
                if flag.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": smax, "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------- workload
class Workload:
    def __init__(self, name: str, lens, shape, seed: int = 0, device="cuda", layout: str = "fragmented"):
        import torch
        self.name, self.shape = name, shape
        self.lens = np.asarray(lens, dtype=np.int64)
        self.table = synth.make_page_table(self.lens, seed=seed, spare_pages=64, layout=layout)
        g = torch.Generator(device=device).manual_seed(seed)
        B, t = len(self.lens), self.table
        self.q = torch.randn(B, shape.num_q_heads, 128, device=device, generator=g).to(torch.bfloat16)
        self.k = torch.empty(t.num_pages, shape.num_kv_heads, 16, 128, dtype=torch.bfloat16, device=device)
        self.v = torch.empty_like(self.k)
        for x in (self.k, self.v):      # chunked to bound the fp32 temporary
            for s in range(0, t.num_pages, 8192):
                e = min(t.num_pages, s + 8192)
                x[s:e] = torch.randn(e - s, *x.shape[1:], device=device, generator=g).to(torch.bfloat16)
        self.indptr = torch.from_numpy(t.indptr).to(device)
        self.indices = torch.from_numpy(t.indices).to(device)
        self.kv_len = torch.from_numpy(t.kv_len).to(device)
        self.out = torch.empty(B, shape.num_q_heads, 128, dtype=torch.float32, device=device)
        self.lse = torch.empty(B, shape.num_q_heads, dtype=torch.float32, device=device)

    @property
    def bytes_kv(self):
        return kv_bytes(self.lens, self.shape)

    @property
    def bytes_algo(self):
        return algo_bytes(self.lens, self.shape)


def make_l4(wl: Workload, flags: int = 0):
    from paper_2512_19179_b200 import l4
    params = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads, flags=flags)
    ws = l4.alloc_workspace(params, wl.table.total_pages)
    return l4, params, ws


def time_steps(wl: Workload, steps: int, warmup: int, mode: str = "early"):
    """Device time of `steps` hot-path steps on the current stream.
    mode "early": one l4_decode_attention call per step (plan a1 inside the split-KV kernel,
    one launch) with L4_DECODE_EARLY_INPUTS: back-to-back calls overlap, the next call plans
    and streams its first work item while the previous one finishes (its inputs are not
    written between steps, the flag's precondition);
    "fused": the same call without the flag (each call starts reading after the previous
    one completed: the isolated-call cost);
    "plan_run": l4_decode_plan + l4_decode_run (two launches); "run": l4_decode_run only,
    reusing one materialised plan (what layers 2..n of a decode iteration do)."""
    import torch
    from paper_2512_19179_b200 import l4 as _l4
    l4, params, ws = make_l4(wl, flags=_l4.L4_DECODE_EARLY_INPUTS if mode == "early" else 0)
    st = torch.cuda.current_stream()

    def step():
        if mode in ("early", "fused"):
            l4.attention_call(params, wl.q, wl.k, wl.v, wl.indptr, wl.indices, wl.kv_len, wl.table.total_pages,
                              wl.out, wl.lse, ws)
            return
        if mode == "plan_run":
            l4.decode_plan(params, wl.kv_len, wl.indptr, wl.table.total_pages, ws)
        l4.decode_run(params, wl.q, wl.k, wl.v, wl.indices, wl.out, wl.lse, ws)

    # a materialised plan for plan_info (and for mode "run")
    l4.decode_plan(params, wl.kv_len, wl.indptr, wl.table.total_pages, ws)
    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    # one event pair around the K steps: an event recorded between two launches would stop
    # the next launch from overlapping the previous one (programmatic dependent launch)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1)
    return total, None, l4.plan_info(ws)


def time_e2e(wl: Workload, steps: int, warmup: int, n_streams: int = 2, out_bf16: bool = False):
    """Same metric through the public API with HOST buffers.  Every step copies its inputs
    (q, kv_len, indptr, indices: packed in one pinned host buffer, one H2D copy) to the device,
    runs l4_decode_attention and copies the fp32 output back (one D2H copy).  Copies run on
    their own streams and everything is double-buffered (inputs, outputs, workspaces, and two
    compute streams), so step i+1's H2D, step i's kernel and step i-1's D2H overlap, and
    consecutive kernels (on alternating streams) overlap each other's tail and head, as in a
    pipelined serving loop; the timed region spans the first H2D to the last D2H."""
    import torch
    from paper_2512_19179_b200 import l4 as _l4
    from paper_2512_19179_b200 import l4 as l4m
    l4, params, ws0 = make_l4(wl)
    if out_bf16:
        params = l4m.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads, out_dtype=l4m.L4_DT_BF16)
    ws = [ws0, torch.zeros_like(ws0)]
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    s_cmps = [torch.cuda.Stream() for _ in range(n_streams)]
    parts = [wl.q, wl.kv_len, wl.indptr, wl.indices]
    offs, off = [], 0
    for t in parts:
        offs.append(off)
        off += (t.numel() * t.element_size() + 255) // 256 * 256
    h_pack = torch.empty(off, dtype=torch.uint8).pin_memory()
    for t, o in zip(parts, offs):
        nb = t.numel() * t.element_size()
        h_pack[o:o + nb].copy_(t.cpu().contiguous().view(-1).view(torch.uint8))
    d_pack = [torch.empty(off, dtype=torch.uint8, device="cuda") for _ in range(2)]

    def views(buf):
        out = []
        for t, o in zip(parts, offs):
            nb = t.numel() * t.element_size()
            out.append(buf[o:o + nb].view(t.dtype).view(t.shape))
        return out
    d_in = [views(d) for d in d_pack]
    odt = torch.bfloat16 if out_bf16 else torch.float32
    d_out = [torch.empty(wl.out.shape, dtype=odt, device="cuda") for _ in range(2)]
    d_lse = [torch.empty_like(wl.lse) for _ in range(2)]
    h_out = [torch.empty(wl.out.shape, dtype=odt).pin_memory() for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in parts)
    d2h = h_out[0].numel() * h_out[0].element_size()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]
    for e in ev_cmp + ev_out:
        e.record(s_cmps[0])

    def step(i):
        b = i % 2
        s_cmp = s_cmps[i % n_streams]
        with torch.cuda.stream(s_h2d):
            s_h2d.wait_event(ev_cmp[b])            # step i-2 finished reading these inputs
            d_pack[b].copy_(h_pack, non_blocking=True)
            ev_in[b].record(s_h2d)
        with torch.cuda.stream(s_cmp):
            s_cmp.wait_event(ev_in[b])
            s_cmp.wait_event(ev_out[b])            # step i-2's output has been copied out
            q, kl, ip, ix = d_in[b]
            l4.attention_call(params, q, wl.k, wl.v, ip, ix, kl, wl.table.total_pages, d_out[b], d_lse[b], ws[b],
                              stream=s_cmp)
            ev_cmp[b].record(s_cmp)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_cmp[b])
            h_out[b].copy_(d_out[b], non_blocking=True)
            ev_out[b].record(s_d2h)

    for i in range(warmup):
        step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_h2d)
    for i in range(steps):
        step(i)
    s_d2h.synchronize()
    s_h2d.wait_stream(s_d2h)
    e1.record(s_h2d)
    e1.synchronize()
    return e0.elapsed_time(e1), h2d, d2h


def cpu_oracle_sample(wl_name: str, budget_s: float = 12.0):
    """The FP64 oracle, as it stands, on a bounded sample of the workload: its requests in
    workload order (cycling through the batch again if one pass takes less than the budget)
    until ~budget_s seconds of oracle time."""
    import torch
    from oracle import attention as oa
    spec = WORKLOADS[wl_name]
    shape = spec["shape"]
    lens = spec["lens"]()
    cores = len(os.sched_getaffinity(0))
    done_tokens, n_req, oracle_time = 0, 0, 0.0
    g = torch.Generator().manual_seed(1234)
    while oracle_time < budget_s:
        b = n_req % len(lens)
        L = int(lens[b])
        table = synth.make_page_table([L], seed=b, spare_pages=0, layout="contiguous")
        q = torch.randn(1, shape.num_q_heads, 128, generator=g).to(torch.bfloat16)
        k = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, generator=g).to(torch.bfloat16)
        v = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, generator=g).to(torch.bfloat16)
        t0 = time.perf_counter()        # input generation is excluded; the oracle call is timed
        oa.paged_decode_attention(q, k, v, table.indptr, table.indices, table.kv_len, shape.num_kv_heads)
        oracle_time += time.perf_counter() - t0
        done_tokens += L
        n_req += 1
    gbs = kv_bytes([done_tokens], shape) / oracle_time / 1e9
    try:
        import threadpoolctl
        blas = max((x.get("num_threads", 1) for x in threadpoolctl.threadpool_info()), default=1)
    except Exception:
        blas = None
    passes = n_req / len(lens)
    return dict(value=round(gbs, 4), unit="GB/s", cores=cores, kind="oracle",
                sample=f"{n_req} requests of {wl_name} in workload order ({passes:.2f} passes over its {len(lens)} "
                       f"requests, {done_tokens} tokens), FP64 NumPy, {oracle_time:.1f} s of oracle time; "
                       f"BLAS threads {blas}", seconds=round(oracle_time, 3),
                tokens=done_tokens, requests=n_req)


# ----------------------------------------------------------------------------- binned vs mixed
def mixed_vs_binned(steps: int, warmup: int):
    """C3 (seed 0): one mixed call vs the same requests split into power-of-4 length
    bins (one call per bin, all on one stream); plus C4 as a long-stage batch."""
    import torch
    res = {}
    shape = synth.SHAPE_LLAMA3_8B
    lens = synth.lengths_c3(0)
    wl = Workload("c3", lens, shape)
    tot, _, info = time_steps(wl, steps, warmup)
    res["c3_mixed"] = dict(gbs=round(wl.bytes_kv / (tot / steps / 1e3) / 1e9, 1), ms=round(tot / steps, 4),
                           items=info.num_items, chunk_pages=info.chunk_pages)
    edges = [0, 1024, 4096, 16384, 65536, 1 << 30]
    t_sum, b_sum, bins = 0.0, 0, []
    del wl
    for lo, hi in zip(edges, edges[1:]):
        sel = lens[(lens >= lo) & (lens < hi)]
        if len(sel) == 0:
            continue
        w = Workload(f"c3[{lo},{hi})", sel, shape)
        t, _, _ = time_steps(w, steps, warmup)
        t_sum += t / steps
        b_sum += w.bytes_kv
        bins.append(dict(lo=lo, hi=hi if hi < (1 << 30) else None, batch=int(len(sel)),
                         gbs=round(w.bytes_kv / (t / steps / 1e3) / 1e9, 1)))
        del w
    res["c3_binned_same_requests"] = dict(gbs=round(b_sum / (t_sum / 1e3) / 1e9, 1), ms=round(t_sum, 4), bins=bins)
    torch.cuda.empty_cache()
    # (iii) stage-shaped binned: for each length class a homogeneous batch (the class's median
    # length) refilled to about the C3 KV volume (<= 1024 requests): what an L4 stage instance sees
    stage_shaped = []
    for b in bins:
        sel = lens[(lens >= b["lo"]) & (lens < (b["hi"] or (1 << 30)))]
        L = int(np.median(sel))
        n = int(min(1024, max(1, round(lens.sum() / L))))
        w = Workload(f"stage[{b['lo']}]", np.full(n, L, dtype=np.int64), shape)
        t, _, _ = time_steps(w, steps, warmup)
        stage_shaped.append(dict(lo=b["lo"], hi=b["hi"], length=L, batch=n,
                                 gbs=round(w.bytes_kv / (t / steps / 1e3) / 1e9, 1)))
        del w
        torch.cuda.empty_cache()
    res["c3_stage_shaped_binned"] = stage_shaped
    w = Workload("c4", synth.lengths_c4(0), synth.SHAPE_LLAMA3_70B)
    t, _, info = time_steps(w, steps, warmup)
    res["c4"] = dict(gbs=round(w.bytes_kv / (t / steps / 1e3) / 1e9, 1), ms=round(t / steps, 4),
                     items=info.num_items, chunk_pages=info.chunk_pages)
    del w
    torch.cuda.empty_cache()
    # SURVEY §8(d) variants: C3 "production-like" (16 long, short median 2048), C2 with a partial
    # last page (L = 1000, the paper's "1000-token"), C2 with an identity page layout
    variants = (("c3_production", synth.lengths_c3_production(0), shape, "fragmented"),
                ("c2_L1000", synth.lengths_c2(length=1000), shape, "fragmented"),
                ("c2_contiguous", synth.lengths_c2(), shape, "contiguous"))
    for name, lens_v, shape_v, layout in variants:
        w = Workload(name, lens_v, shape_v, layout=layout)
        t, _, _ = time_steps(w, steps, warmup)
        res[name] = dict(gbs=round(w.bytes_kv / (t / steps / 1e3) / 1e9, 1), ms=round(t / steps, 4),
                         sum_len=int(np.sum(lens_v)), layout=layout)
        del w
        torch.cuda.empty_cache()
    return res


def heterogeneity_slowdown(steps: int, warmup: int):
    """Fig. 2 (`fig:interference`) analogue on our kernel: batch 512,
    k long requests among short ones (1000 vs 50000 and 200 vs 10000) against a homogeneous
    batch with the same batch size and the same total tokens.  The paper measured 1.1-2.1x
    slowdowns on H100 with FlashAttention / FlashInfer / Triton."""
    import torch
    out = []
    for short, long in ((1000, 50000), (200, 10000)):
        for k in (1, 8, 32):
            mixed = synth.lengths_fig2(512, k, short, long)
            homo = np.full(512, int(round(mixed.sum() / 512)), dtype=np.int64)
            row = dict(short=short, long=long, n_long=k, sum_len=int(mixed.sum()))
            for name, lens in (("mixed", mixed), ("homogeneous", homo)):
                w = Workload(name, lens, synth.SHAPE_LLAMA3_8B)
                t, _, _ = time_steps(w, steps, warmup)
                row[name + "_us"] = round(t / steps * 1e3, 2)
                row[name + "_gbs"] = round(w.bytes_kv / (t / steps / 1e3) / 1e9, 1)
                del w
                torch.cuda.empty_cache()
            row["slowdown"] = round(row["mixed_us"] / row["homogeneous_us"], 3)
            out.append(row)
    return out


def short_batches(steps: int, warmup: int):
    """Homogeneous batches of short requests at the largest single-launch batch (B = 1024,
    Llama-3-8B and -70B shapes): the per-item overheads the quad units remove."""
    import torch
    out = []
    for shape, L in ((synth.SHAPE_LLAMA3_8B, 64), (synth.SHAPE_LLAMA3_8B, 200), (synth.SHAPE_LLAMA3_8B, 530),
                     (synth.SHAPE_LLAMA3_70B, 64), (synth.SHAPE_LLAMA3_70B, 200)):
        w = Workload(f"short{L}", np.full(1024, L, dtype=np.int64), shape)
        t, _, _ = time_steps(w, steps, warmup)
        out.append(dict(shape=shape.name, length=L, batch=1024, us=round(t / steps * 1e3, 2),
                        gbs=round(w.bytes_kv / (t / steps / 1e3) / 1e9, 1)))
        del w
        torch.cuda.empty_cache()
    return out


def migration_bandwidth(reps: int = 10):
    """l4_migrate of one request at the Llama-3-8B shape with all 32 layers:
    a 2048-token request = 128 pages x 32 layers x (K, V) = 256 MiB.  Loopback on one GPU
    (HBM -> HBM: every byte read and written once); over NVLink the same kernel writes to
    IPC-mapped peer pools.  Reported: the copy kernel alone (l4_copy_pages, `reps` launches
    between one event pair), the whole l4_migrate call (host allocation + launch, per call),
    and torch's device copy of the same byte count as the loopback reference."""
    import torch
    from paper_2512_19179_b200 import l4
    layers, pages, n = 32, 2048, 128
    k = torch.empty(layers, pages, 8, 16, 128, dtype=torch.bfloat16, device="cuda")
    v = torch.empty_like(k)
    k2, v2 = torch.empty_like(k), torch.empty_like(v)
    src, dst = l4.kv_view(k, v, num_layers=layers), l4.kv_view(k2, v2, num_layers=layers)
    sp = np.random.default_rng(0).permutation(pages)[:n]
    dp = np.random.default_rng(1).permutation(pages)[:n]
    nbytes = n * layers * 2 * src.page_bytes

    def timed(fn, r):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(r):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / r

    t_kernel = timed(lambda: l4.copy_pages(src, sp, dst, dp), reps)
    times = []
    for i in range(reps + 2):
        pool = l4.PagePool(pages)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        l4.migrate(src, sp, dst, pool)
        e1.record()
        e1.synchronize()
        if i >= 2:
            times.append(e0.elapsed_time(e1))
    t_call = float(np.median(times))
    a_ = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    b_ = torch.empty_like(a_)
    t_torch = timed(lambda: b_.copy_(a_), reps)
    del k, v, k2, v2, a_, b_
    torch.cuda.empty_cache()
    return dict(request_tokens=n * 16, layers=layers, bytes=int(nbytes),
                kernel_ms=round(t_kernel, 4), kernel_gbs_moved=round(nbytes / (t_kernel / 1e3) / 1e9, 1),
                kernel_gbs_hbm_traffic=round(2 * nbytes / (t_kernel / 1e3) / 1e9, 1),
                call_ms=round(t_call, 4), call_gbs_moved=round(nbytes / (t_call / 1e3) / 1e9, 1),
                torch_copy_same_bytes_ms=round(t_torch, 4),
                note="loopback src->dst on one GPU; HBM traffic = read + write; 4096 32 KB slices")


def fitted_qoe_d(layers: int = 32):
    """Eq. (1)'s D fitted on this kernel's measured step times (NEXT#3, the newest committed
    profiles/qoe_fit_*.json, one layer) scaled to a `layers`-layer decode step; else None (the
    partition then uses the roofline D, Z15)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "qoe_fit_r*.json")))
    if not files:
        return None, "roofline (synth.roofline_qoe_d, Z15)"
    d = json.load(open(files[-1]))["D"]
    return tuple(float(x) * layers for x in d), f"fitted ({os.path.relpath(files[-1], ROOT)}) x {layers} layers"


def partition_speed():
    """l4_partition (host C++) over 10,000 ShareGPT-like requests (lengths up
    to 128K) at E = 4, 8, 16 instances; the paper plans E = 16 in 0.06 s."""
    from paper_2512_19179_b200 import l4
    I, O = synth.requests_sharegpt_like(seed=1, n=10000)
    D = synth.roofline_qoe_d()
    res = {}
    for E in (4, 8, 16):
        t = time.perf_counter()
        stages, obj = l4.partition(I, O, E, D, 7e11, 131072, mode=0)
        dt = time.perf_counter() - t
        t = time.perf_counter()
        l4.partition(I, O, E, D, 7e11, 131072, mode=0, algorithm=l4.PART_TWO_PHASE)
        dt2 = time.perf_counter() - t
        res[f"E{E}"] = dict(exact_dp_ms=round(dt * 1e3, 3), two_phase_ms=round(dt2 * 1e3, 3), stages=stages,
                            objective=obj)
    return res


def partition_oracle_speed():
    """The partition oracle (pure Python, one core) on the same M6 inputs (cpu_baseline leg)."""
    from oracle import partition as op
    I, O = synth.requests_sharegpt_like(seed=1, n=10000)
    D = synth.roofline_qoe_d()
    res = {}
    for E in (4, 16):
        t = time.perf_counter()
        op.plan_dp(I, O, E, D, 7e11, 131072, mode=0)
        res[f"E{E}_s"] = round(time.perf_counter() - t, 3)
    return res


# ----------------------------------------------------------------------------- pipeline (N > 1)
def run_pipeline_arm(stages, steps, warmup, rank, world, device, per_rank=256, seed=0, shape=None, precopy_lead=0,
                     policy="least_loaded", rebalance_every=0, e2e=False):
    """C5: the length-aware pipeline on `world` GPUs.  Every step each rank runs the hot path
    (plan + split-KV kernel) on its resident batch, then the replicated control plane advances
    (tokens appended, handovers, retirements, arrivals) and KV pages of handed-over requests
    move between ranks (l4_pack_pages -> NCCL send/recv -> l4_unpack_pages).
    With e2e=True every step also copies its batch's query rows in from pinned host memory and
    its attention output back to pinned host memory (the end-to-end variant).
    Returns per-rank totals (device time measured with CUDA events on the compute stream)."""
    import torch
    import torch.distributed as dist
    from paper_2512_19179_b200 import l4, pipeline
    shape = shape or synth.SHAPE_LLAMA3_8B
    sim = pipeline.ClusterSim(stages, concurrency=world * per_rank, seed=seed, precopy_lead=precopy_lead,
                              policy=policy, rebalance_every=rebalance_every)
    budget_pages = sim.token_budget // 16 * 5 // 4 + 2 * sim.batch_cap
    rt = pipeline.RankRuntime(sim, rank, budget_pages, shape, pipeline.DeviceOps(shape, device, seed + rank))
    if os.environ.get("L4_PIPE_TRANSPORT", "nccl") == "ipc" and world > 1:
        # one-sided transport: peers' pools mapped through CUDA IPC, metadata over a CPU group
        cpu_group = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else None
        rt.ops.setup_ipc(rt.pool, rank, world, cpu_group)
    cap = sim.batch_cap
    g = torch.Generator(device=device).manual_seed(seed + 100 + rank)
    q = torch.randn(cap, shape.num_q_heads, 128, device=device, generator=g).to(torch.bfloat16)
    out = torch.empty(cap, shape.num_q_heads, 128, dtype=torch.float32, device=device)
    lse = torch.empty(cap, shape.num_q_heads, dtype=torch.float32, device=device)
    if e2e:
        # double-buffered query rows / outputs; copies on their own streams overlap the kernels
        h_q = q.cpu().pin_memory()
        h_out = [torch.empty(out.shape, dtype=out.dtype).pin_memory() for _ in range(2)]
        q_buf, out_buf = [q, torch.empty_like(q)], [out, torch.empty_like(out)]
        s_in, s_out = torch.cuda.Stream(device=device), torch.cuda.Stream(device=device)
        ev_k = [torch.cuda.Event() for _ in range(2)]
        ev_in = [torch.cuda.Event() for _ in range(2)]
        for e in ev_k:
            e.record(torch.cuda.current_stream())
    p_max = l4.make_params(cap, shape.num_q_heads, shape.num_kv_heads)
    ws = l4.alloc_workspace(p_max, budget_pages)
    pool = rt.pool
    tot = dict(kv_bytes=0, tokens=0, steps=0, mig_bytes=0, mig_count=0, busy_ms=0.0, req_steps=0, lat_ms_x_req=0.0)
    evs = []
    st = torch.cuda.current_stream()
    t_start = t_end = None
    for it in range(warmup + steps):
        timed = it >= warmup
        if it == warmup:
            torch.cuda.synchronize()
            dist.barrier()
            t_start = torch.cuda.Event(enable_timing=True)
            t_start.record(st)
        kv_len, indptr = rt.device_batch()
        B = int(kv_len.shape[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        if B > 0:
            d_len, d_ptr = rt.ops.h2d.put(kv_len, indptr)
            params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads)
            qx, ox = q, out
            if e2e:
                bi = it % 2
                qx, ox = q_buf[bi], out_buf[bi]
                s_in.wait_event(ev_k[bi])                 # the kernel two steps back read this buffer
                if it == warmup:
                    s_in.wait_event(t_start)              # the first timed copy starts inside the region
                with torch.cuda.stream(s_in):
                    qx[:B].copy_(h_q[:B], non_blocking=True)
                    ev_in[bi].record(s_in)
                st.wait_event(ev_in[bi])
            l4.attention_call(params, qx[:B], pool["k"], pool["v"], d_ptr, rt.table, d_len, int(rt.table.numel()),
                              ox[:B], lse[:B], ws)
            if e2e:
                ev_k[bi].record(st)
                s_out.wait_event(ev_k[bi])
                with torch.cuda.stream(s_out):
                    h_out[bi][:B].copy_(ox[:B], non_blocking=True)
                if timed:
                    tot["h2d"] = tot.get("h2d", 0) + B * shape.num_q_heads * 128 * 2 + 8 * B
                    tot["d2h"] = tot.get("d2h", 0) + B * shape.num_q_heads * 128 * 4
        e1.record(st)
        ev = sim.step()
        before = rt.stats["migrated_bytes"]
        rt.apply(ev, dist)
        if timed:
            evs.append((e0, e1, B))
            tot["kv_bytes"] += int(4 * shape.num_kv_heads * 128 * int(kv_len.sum()))
            tot["launches"] = tot.get("launches", 0) + (1 if B > 0 else 0)
            tot["tokens"] += B
            tot["steps"] += 1
            tot["mig_bytes"] += rt.stats["migrated_bytes"] - before
            tot["mig_count"] += sum(1 for m in ev.migrations if m[1] == rank)
    t_end = torch.cuda.Event(enable_timing=True)
    if e2e:
        st.wait_stream(s_out)                             # the last output copy is inside the timed region
    t_end.record(st)
    torch.cuda.synchronize()
    for e0, e1, B in evs:
        dt = e0.elapsed_time(e1)
        tot["busy_ms"] += dt
        tot["lat_ms_x_req"] += dt * B
        tot["req_steps"] += B
    tot["elapsed_ms"] = t_start.elapsed_time(t_end)
    tot["launches"] = tot.get("launches", 0) + rt.stats["launches"]
    for k_ in ("precopy_pages", "stop_pages", "single_pages"):
        tot[k_] = rt.stats[k_]
    tot["fingerprint"] = sim.fingerprint()
    if hasattr(rt.ops, "close_ipc"):
        rt.ops.close_ipc()
    tot["stage_cv"] = sim.stage_cv()
    tot["stages"] = stages
    return tot


def pipeline_line(args, world, rank, local):
    import torch
    import torch.distributed as dist
    from paper_2512_19179_b200 import pipeline
    device = torch.device("cuda", local)
    cdev = device if dist.get_backend() == "nccl" else torch.device("cpu")   # collectives' device
    peak, peak_src = load_peaks()
    qoe_d, qoe_src = fitted_qoe_d()
    stages, obj = pipeline.plan_stages(world, seed=0, qoe_d=qoe_d)
    rr = [(0, stages[-1][1], world)]                       # length-agnostic: one stage of all instances
    res = {}
    dist.barrier()                                          # first collective on the group
    # warm up the NCCL P2P connections between every pair of ranks (handovers go to the next
    # stage, rebalancing stays inside a stage) outside the timed region
    ops = []
    for peer in range(world):
        if peer != rank:
            ops.append(dist.P2POp(dist.isend, torch.ones(1, device=cdev), peer))
            ops.append(dist.P2POp(dist.irecv, torch.empty(1, device=cdev), peer))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    torch.cuda.synchronize()
    dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    for name, st in (("l4", stages), ("round_robin", rr), ("l4_e2e", stages)):
        # L4 arm: bid-ask receivers + intra-stage rebalancing and live (two-round)
        # migration with an 8-token pre-copy lead; baseline: one length-agnostic stage,
        # round-robin placement
        l4arm = name != "round_robin"
        t = run_pipeline_arm(st, args.steps, args.warmup, rank, world, device,
                             precopy_lead=8 if l4arm else 0, policy="bidask" if l4arm else "round_robin",
                             rebalance_every=10 if l4arm else 0, e2e=name == "l4_e2e")
        if name == "l4":
            clk = clocks.stop()
        vec = torch.tensor([t["kv_bytes"], t["tokens"], t["mig_bytes"], t["mig_count"], t["req_steps"],
                            t["lat_ms_x_req"], t["launches"], t["precopy_pages"], t["stop_pages"],
                            t["single_pages"], t.get("h2d", 0), t.get("d2h", 0), t["busy_ms"]],
                           dtype=torch.float64, device=cdev)
        dist.all_reduce(vec, op=dist.ReduceOp.SUM)
        tm = torch.tensor([t["elapsed_ms"], t["busy_ms"]], dtype=torch.float64, device=cdev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        fp = torch.tensor([t["fingerprint"] & 0x7FFFFFFF], dtype=torch.int64, device=cdev)
        fps = [torch.zeros_like(fp) for _ in range(world)]
        dist.all_gather(fps, fp)
        assert all(int(x) == int(fp) for x in fps), "replicated control plane diverged"
        elapsed = float(tm[0])
        res[name] = dict(kv_gbs=float(vec[0]) / (elapsed / 1e3) / 1e9, tokens_per_s=float(vec[1]) / (elapsed / 1e3),
                         elapsed_ms=elapsed, max_busy_ms=float(tm[1]), migrated_bytes=int(vec[2]),
                         migrations=int(vec[3]), mean_step_latency_ms=float(vec[5]) / max(1.0, float(vec[4])),
                         stage_cv=[round(x, 4) for x in t["stage_cv"]],
                         launches=int(vec[6]), precopy_pages=int(vec[7]), stop_round_pages=int(vec[8]),
                         single_round_pages=int(vec[9]), h2d_bytes=int(vec[10]), d2h_bytes=int(vec[11]),
                         sum_busy_ms=float(vec[12]), kv_bytes=float(vec[0]),
                         stages=[list(x) for x in st])
    if rank != 0:
        return None
    l4r = res["l4"]
    mig_gbs = None
    line = {
        "metric": METRIC, "value": round(l4r["kv_gbs"], 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(l4r["elapsed_ms"] / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "c5-pipeline", "desc": "BASELINE configs[4]: length-aware pipeline, "
                   f"{world} instances (1 GPU each), Llama-3-8B attention shape, ShareGPT-like closed loop, "
                   f"{256} resident requests per instance, 1.2M-token KV budget per instance",
                   "stages": l4r["stages"], "partition_objective": obj, "qoe_d": list(qoe_d) if qoe_d else None,
                   "qoe_d_source": qoe_src,
                   "parallelism": f"length-aware pipeline over {world} GPUs (l4_partition); KV migration "
                                  + ("one-sided over CUDA IPC (l4_copy_pages into peers' pools)"
                                     if os.environ.get("L4_PIPE_TRANSPORT", "nccl") == "ipc"
                                     else "over NCCL P2P (l4_pack_pages / l4_unpack_pages)"),
                   "l2": "inputs larger than L2; no flush"},
        "tokens_per_s": round(l4r["tokens_per_s"], 1),
        "pct_hbm_peak": round(100.0 * l4r["kv_gbs"] / (world * peak), 2),
        "pipeline": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                     for k, v in res.items()},
        "gpu_launches": int(l4r["launches"]),
        "clocks": clk,
    }
    # dominant kernel: the per-step decode launch of every rank (algorithmic KV bytes over the
    # summed event time of those launches, all ranks)
    ach = l4r["kv_bytes"] / (l4r["sum_busy_ms"] / 1e3) / 1e9 if l4r["sum_busy_ms"] > 0 else None
    line["roofline"] = {"bound": "hbm", "kernel": "decode_kernel<G, fused> (per-rank l4_decode_attention)",
                        "achieved": round(ach, 1) if ach else None, "peak": peak, "unit": "GB/s",
                        "frac": round(ach / peak, 4) if ach else None, "traffic": None, "peak_source": peak_src,
                        "note": "KV bytes only (q/out/ids not counted); per-GPU"}
    e = res["l4_e2e"]
    line["e2e"] = {"value": round(e["kv_gbs"], 1), "unit": "GB/s",
                   "h2d_bytes_per_step": int(e["h2d_bytes"] / max(1, args.steps)),
                   "d2h_bytes_per_step": int(e["d2h_bytes"] / max(1, args.steps)),
                   "note": "the L4 arm again with every step's query rows copied in from pinned host memory and "
                           "its attention output copied back (bytes summed over ranks)"}
    return line


# ----------------------------------------------------------------------------- main
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    name = args.workload
    spec = WORKLOADS[name]
    budget = max(2.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_oracle_sample(name, budget_s=budget / 4)
    vals, samples = [], None
    for _ in range(args.steps):
        r = cpu_oracle_sample(name, budget_s=budget)
        vals.append(r["value"])
        samples = r
    v = float(np.mean(vals))
    full_bytes = kv_bytes(spec["lens"](), spec["shape"])
    ms_full = full_bytes / (v * 1e9) * 1e3          # the oracle's time for one whole step, at the sampled rate
    line = dict(impl="reference", metric=METRIC, value=round(v, 4), unit="GB/s", n_gpus=args.gpus,
                steps=args.steps, warmup=args.warmup, ms_per_step=round(ms_full, 3), higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=name, desc=spec["desc"], batch=len(spec["lens"]()),
                            kv_bytes_per_step=full_bytes),
                cpu_baseline=dict(value=round(v, 4), unit="GB/s", cores=samples["cores"], kind="oracle",
                                  sample=samples["sample"]),
                e2e=dict(value=round(v, 4), unit="GB/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="l4", choices=["l4", "reference"])
    ap.add_argument("--no-extra", action="store_true", help="skip mixed-vs-binned / C4 sub-measurements")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of the pipeline")
    ap.add_argument("--pipeline", action="store_true", help="run the C5 pipeline harness even at N = 1")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    import torch
    ws, rank, local = dist_env()
    # development only: L4_FORCE_DEVICE pins every rank to one GPU and L4_PIPE_BACKEND=gloo
    # swaps NCCL for gloo (host-staged transport), so the N-rank harness runs on one B200
    local = int(os.environ.get("L4_FORCE_DEVICE", local))
    backend = os.environ.get("L4_PIPE_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if (ws > 1 and not args.replicas) or args.pipeline:
        if ws == 1:
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            torch.distributed.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                                                 world_size=1, device_id=torch.device("cuda", local))
        line = pipeline_line(args, ws, rank, local)
        if rank == 0:
            print(json.dumps(line), flush=True)
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
        return 0
    peak, peak_src = load_peaks()
    spec = WORKLOADS[args.workload]
    wl = Workload(args.workload, spec["lens"](), spec["shape"], seed=rank)
    from paper_2512_19179_b200 import l4

    # warm-up + build plan once for run-only timing
    time_steps(wl, 2, args.warmup)
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    total_ms, per, info = time_steps(wl, args.steps, 1)             # the step: one fused launch
    clk = clocks.stop()
    iso_ms, _, _ = time_steps(wl, args.steps, 1, mode="fused")
    pr_ms, _, _ = time_steps(wl, args.steps, 1, mode="plan_run")
    run_ms, _, _ = time_steps(wl, args.steps, 1, mode="run")
    if ws > 1:
        t = torch.tensor([total_ms, run_ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.barrier()
        total_ms, run_ms = float(t[0]), float(t[1])
    ms_step = total_ms / args.steps
    value = ws * wl.bytes_kv / (ms_step / 1e3) / 1e9
    # roofline of the dominant kernel: the step is one launch of the fused decode_kernel, so its
    # average launch duration is the event time over the timed region / steps (consecutive
    # launches overlap by the early start: this is the steady-state per-launch time)
    launch_avg = total_ms / args.steps
    run_avg = run_ms / args.steps
    achieved = wl.bytes_algo / (launch_avg / 1e3) / 1e9
    # a pipelined loop: the timed region holds one fill (first H2D) and one drain (last D2H), so
    # it runs at least 50 steps to keep those to a few percent of the total
    e2e_steps = max(50, args.steps)
    e2e_ms, h2d, d2h = time_e2e(wl, e2e_steps, max(5, args.warmup))
    e2e_step = e2e_ms / e2e_steps
    extra = {}
    if rank == 0 and ws == 1 and not args.no_extra:
        extra = mixed_vs_binned(max(5, args.steps // 2), 3)
        extra["fig2_heterogeneity"] = heterogeneity_slowdown(max(5, args.steps // 2), 3)
        extra["short_batches"] = short_batches(max(5, args.steps // 2), 3)
        extra["migration"] = migration_bandwidth()
        extra["partition_m6"] = partition_speed()
    rceil, rceil_src = read_ceiling()
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(args.workload, budget_s=12.0)
    if rank != 0:
        return 0
    traffic, traffic_src = measured_traffic(args.workload)
    line = {
        "metric": METRIC,
        "value": round(value, 1),
        "unit": "GB/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 5),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic",
        "config": {"workload": args.workload, "desc": spec["desc"], "batch": int(len(wl.lens)),
                   "sum_kv_len": int(wl.lens.sum()), "kv_bytes_per_step": wl.bytes_kv,
                   "num_q_heads": wl.shape.num_q_heads, "num_kv_heads": wl.shape.num_kv_heads, "head_dim": 128,
                   "page_size": 16, "page_layout": "fragmented (seeded permutation)",
                   "l2": "inputs larger than L2 (KV working set >> 126 MB); no flush",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single instance",
                   "plan": {"items": info.num_items, "chunk_pages": info.chunk_pages, "ctas": info.num_ctas},
                   "call": "l4_decode_attention (plan + split-KV + combine in one kernel launch), "
                           "flags=L4_DECODE_EARLY_INPUTS, back-to-back steps"},
        "tokens_per_s": round(ws * len(wl.lens) / (ms_step / 1e3), 1),
        "tokens_per_s_depth_normalised": {
            "value": round(ws * len(wl.lens) / (ms_step / 1e3) / (80 if wl.shape.num_q_heads == 64 else 32), 1),
            "layers": 80 if wl.shape.num_q_heads == 64 else 32,
            "note": "SURVEY 8(d): B / (n_layers x t_call), attention time only (Llama-3-8B 32 / -70B 80 layers)"},
        "pct_hbm_peak": round(100.0 * value / (ws * peak), 2),
        "roofline": {"bound": "hbm", "kernel": "decode_kernel<G, fused> (l4_decode_attention, "
                                               "L4_DECODE_EARLY_INPUTS)",
                     "achieved": round(achieved, 1),
                     "peak": peak, "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": traffic,
                     "traffic_source": traffic_src,
                     "peak_source": peak_src, "launch_ms": round(launch_avg, 5),
                     "bytes_per_launch": wl.bytes_algo,
                     "frac_of_nominal_8TBs": round(achieved / 8000.0, 4),
                     "read_ceiling_gbs": rceil,
                     "frac_of_read_ceiling": round(achieved / rceil, 4) if rceil else None,
                     "read_ceiling_source": rceil_src},
        "isolated_call": {"note": "l4_decode_attention without L4_DECODE_EARLY_INPUTS: each call starts "
                                  "reading after the previous one completed",
                          "ms_per_step": round(iso_ms / args.steps, 5),
                          "gbs": round(wl.bytes_kv / (iso_ms / args.steps / 1e3) / 1e9, 1),
                          "roofline_frac": round(wl.bytes_algo / (iso_ms / args.steps / 1e3) / 1e9 / peak, 4)},
        "two_launch_path": {"note": "l4_decode_plan + l4_decode_run per step (materialised plan)",
                            "ms_per_step": round(pr_ms / args.steps, 5),
                            "gbs": round(wl.bytes_kv / (pr_ms / args.steps / 1e3) / 1e9, 1),
                            "run_only_ms": round(run_avg, 5)},
        "amortized_32_layers": {"note": "one materialised plan per decode iteration reused by 32 layers: "
                                        "plan + 32 x run",
                                "gbs": round(32 * wl.bytes_kv / ((pr_ms / args.steps - run_avg + 32 * run_avg) / 1e3)
                                             / 1e9, 1)},
        "e2e": {"value": round(ws * wl.bytes_kv / (e2e_step / 1e3) / 1e9, 1), "unit": "GB/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_step, 5)},
        "gpu_launches": args.steps * (1 if len(wl.lens) <= 1024 else 2),
        "clocks": clk,
    }
    if cpu:
        line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if not args.no_extra:
            line["cpu_baseline"]["partition_m6_oracle"] = partition_oracle_speed()
    if extra:
        line["extra"] = extra
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
