#!/usr/bin/env python3
"""bench.py — L4 hot path on B200: decode-attention KV GB/s (% of HBM peak), mixed vs binned;
tokens/s of the length-aware pipeline at 1/2/4/8 GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3|c2|c4] [--impl l4|reference]

N = 1 (default).  A step is one pass of the hot path over one synthetic batch: one
l4_decode_attention call = the length-binned work-list build (a1, run by every CTA in shared
memory) + the split-KV kernel with its fused LSE combine (a2 + a3), in ONE launch: one decode
iteration of one layer.  The workload is BASELINE configs[2] (C3, the metric's "mixed" batch:
Llama-3-8B shape, 256 ShareGPT-like requests of 100..128K tokens); C4, C2 and the length-binned
batches are extra lines, each with its own roofline object.
  value   algorithmic KV bytes per step / device step time, plain calls (no early-input
          overlap) back to back over 4 rotating copies of every input (q, K/V pools, page
          table; each copy >> 126 MB L2), inputs resident in HBM.
  e2e     the same metric through the public API with HOST buffers: every step copies its
          inputs (q, kv_len, indptr, indices) H2D from pinned memory and its output D2H; the
          step sequence is captured once in a CUDA graph and replayed (host cost per step is
          reported).
  roofline.configs  per-workload kernel-alone numbers: median of >= 30 single calls, each after
          an L2 flush (a 2 x L2 write), bracketed by CUDA events.

N > 1: `python bench.py --gpus N` re-executes itself under torch.distributed.run (one process per
GPU, NCCL); every rank is one serving instance of the length-aware pipeline (BASELINE configs[4]):
l4_partition assigns ranks to length stages, each rank decodes its resident batch every step and
KV pages of requests that outgrow their stage move to the next stage's rank.  value = aggregate
KV GB/s over all ranks (weak scaling: 256 resident requests per instance); time = max over ranks.

--impl reference: the FP64 CPU oracle (oracle/attention.py), as it stands, on a bounded sample
of the same workload — the reference arm for this tier (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOADS = {
    "c1": dict(desc="BASELINE configs[0]: 8q/2kv, d128, batch 4 with KV lengths {16,64,256,1024} (parity case)",
               shape=synth.SHAPE_C1, lens=lambda: synth.lengths_c1()),
    "c2": dict(desc="BASELINE configs[1]: Llama-3-8B attention (32q/8kv, d128), bf16, batch 250, uniform 1K contexts",
               shape=synth.SHAPE_LLAMA3_8B, lens=lambda: synth.lengths_c2()),
    "c3": dict(desc="BASELINE configs[2]: Llama-3-8B shape, batch 256, ShareGPT-like skewed 100..128K (seed 0), "
                    "mixed batch", shape=synth.SHAPE_LLAMA3_8B, lens=lambda: synth.lengths_c3(0)),
    "c4": dict(desc="BASELINE configs[3]: Llama-3-70B attention (64q/8kv), long-context batch 32, 32K..128K (seed 0)",
               shape=synth.SHAPE_LLAMA3_70B, lens=lambda: synth.lengths_c4(0)),
    # homogeneous short-request batches (extra lines; --workload for profiling runs)
    "short64": dict(desc="B = 1024 x 64 tokens, Llama-3-8B shape (short-stage batch)", shape=synth.SHAPE_LLAMA3_8B,
                    lens=lambda: np.full(1024, 64, dtype=np.int64)),
    "short200": dict(desc="B = 1024 x 200 tokens, Llama-3-8B shape (short-stage batch)", shape=synth.SHAPE_LLAMA3_8B,
                     lens=lambda: np.full(1024, 200, dtype=np.int64)),
}


def _stage_lengths(lo: int, hi: int):
    """C3's length class [lo, hi) refilled: a homogeneous batch of the class's median length with
    about C3's KV volume (<= 1024 requests) — the batch an L4 stage instance sees."""
    lens = synth.lengths_c3(0)
    sel = lens[(lens >= lo) & (lens < hi)]
    L = int(np.median(sel))
    return np.full(int(min(1024, max(1, round(lens.sum() / L)))), L, dtype=np.int64)


STAGE_EDGES = [0, 1024, 4096, 16384, 65536, 1 << 30]
for _lo, _hi in zip(STAGE_EDGES, STAGE_EDGES[1:]):
    WORKLOADS[f"stage{_lo}"] = dict(desc=f"C3 length class [{_lo}, {_hi}) refilled (stage-shaped binned batch)",
                                    shape=synth.SHAPE_LLAMA3_8B, lens=(lambda lo=_lo, hi=_hi: _stage_lengths(lo, hi)))
for _L in (530,):
    WORKLOADS[f"short{_L}"] = dict(desc=f"B = 1024 x {_L} tokens, Llama-3-8B shape", shape=synth.SHAPE_LLAMA3_8B,
                                   lens=(lambda L=_L: np.full(1024, L, dtype=np.int64)))
for _L in (64, 200):
    WORKLOADS[f"short70b_{_L}"] = dict(desc=f"B = 1024 x {_L} tokens, Llama-3-70B shape", shape=synth.SHAPE_LLAMA3_70B,
                                       lens=(lambda L=_L: np.full(1024, L, dtype=np.int64)))
METRIC = "decode-attn KV GB/s (% HBM peak), mixed vs binned; tokens/s at 1/2/4/8 GPUs"
L2_BYTES = 126 * (1 << 20)


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy, read+write)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def read_ceiling():
    """HBM read ceiling measured on this pool by the development probe (scripts/readbw.py,
    committed as profiles/readbw_r*.json), for context: the kernel only reads; the roofline
    peak stays MEASURED_PEAKS.json's copy figure."""
    import glob
    best = None
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "readbw_r*.json"))):
        try:
            d = json.load(open(f))
        except ValueError:
            continue
        vals = [v for k, v in d.items() if not k.startswith("copy") and isinstance(v, (int, float))]
        if vals:
            best = (float(max(vals)), os.path.relpath(f, ROOT))
    return best if best else (None, None)


def measured_traffic(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one decode_kernel launch of `workload` from
    the newest committed ncu --set full summary (profiles/r*_traffic.json), or (None, None)."""
    import glob
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")), reverse=True):
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
    """One synthetic batch resident in HBM, with `copies` rotating copies of every input (q, the
    K/V pools, the page table), so consecutive steps never hit data the previous step left in L2."""

    def __init__(self, name: str, lens, shape, seed: int = 0, device="cuda", layout: str = "fragmented",
                 copies: int = 1):
        import torch
        self.name, self.shape = name, shape
        self.lens = np.asarray(lens, dtype=np.int64)
        self.table = synth.make_page_table(self.lens, seed=seed, spare_pages=64, layout=layout)
        g = torch.Generator(device=device).manual_seed(seed)
        B, t = len(self.lens), self.table
        q = torch.randn(B, shape.num_q_heads, 128, device=device, generator=g).to(torch.bfloat16)
        k = torch.empty(t.num_pages, shape.num_kv_heads, 16, 128, dtype=torch.bfloat16, device=device)
        v = torch.empty_like(k)
        for x in (k, v):      # chunked to bound the fp32 temporary
            for s in range(0, t.num_pages, 8192):
                e = min(t.num_pages, s + 8192)
                x[s:e] = torch.randn(e - s, *x.shape[1:], device=device, generator=g).to(torch.bfloat16)
        ip = torch.from_numpy(t.indptr).to(device)
        ix = torch.from_numpy(t.indices).to(device)
        kl = torch.from_numpy(t.kv_len).to(device)
        self.sets = [(q, k, v, ip, ix, kl)]
        for _ in range(copies - 1):
            self.sets.append(tuple(x.clone() for x in self.sets[0]))
        self.out = torch.empty(B, shape.num_q_heads, 128, dtype=torch.float32, device=device)
        self.lse = torch.empty(B, shape.num_q_heads, dtype=torch.float32, device=device)

    q = property(lambda self: self.sets[0][0])
    k = property(lambda self: self.sets[0][1])
    v = property(lambda self: self.sets[0][2])
    indptr = property(lambda self: self.sets[0][3])
    indices = property(lambda self: self.sets[0][4])
    kv_len = property(lambda self: self.sets[0][5])

    @property
    def bytes_kv(self):
        return kv_bytes(self.lens, self.shape)

    @property
    def bytes_algo(self):
        return algo_bytes(self.lens, self.shape)

    @property
    def input_bytes(self):
        return sum(x.numel() * x.element_size() for x in self.sets[0])


def make_l4(wl: Workload, flags: int = 0):
    from paper_2512_19179_b200 import l4
    params = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads, flags=flags)
    ws = l4.alloc_workspace(params, wl.table.total_pages)
    return l4, params, ws


def _call(l4, params, wl, i, ws, stream=None):
    q, k, v, ip, ix, kl = wl.sets[i % len(wl.sets)]
    l4.attention_call(params, q, k, v, ip, ix, kl, wl.table.total_pages, wl.out, wl.lse, ws, stream)


def steady_ms(wl: Workload, steps: int, warmup: int, early: bool = False, early_plan: bool = False):
    """Device time per step of `steps` back-to-back l4_decode_attention calls (one event pair
    around them, rotating input copies).  early=False: plain calls (each call starts reading
    after the previous one completed, as after a kernel that writes q); early=True:
    L4_DECODE_EARLY_INPUTS (the next call plans and streams its first item under the previous
    call's tail); early_plan=True: L4_DECODE_EARLY_PLAN (only the planner's page-table reads run
    under the previous call's tail).  An event between two launches would stop that overlap,
    hence one pair."""
    import torch
    from paper_2512_19179_b200 import l4 as _l4
    flags = _l4.L4_DECODE_EARLY_INPUTS if early else (_l4.L4_DECODE_EARLY_PLAN if early_plan else 0)
    l4, params, ws = make_l4(wl, flags=flags)
    st = torch.cuda.current_stream()
    for i in range(warmup):
        _call(l4, params, wl, i, ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(steps):
        _call(l4, params, wl, i, ws)
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def per_layer_ms(wl: Workload, steps: int, warmup: int, layers: int):
    """A decode step of a `layers`-layer model: one l4_decode_plan (the work list depends only on
    the page table, shared by every layer) and `layers` l4_decode_run calls over rotating input
    copies (each layer reads its own K/V); device time per layer (one event pair around `steps`
    steps)."""
    import torch
    l4, params, ws = make_l4(wl)

    def step():
        q, k, v, ip, ix, kl = wl.sets[0]
        l4.decode_plan(params, kl, ip, wl.table.total_pages, ws)
        for j in range(layers):
            q, k, v, ip, ix, kl = wl.sets[j % len(wl.sets)]
            l4.decode_run(params, q, k, v, ix, wl.out, wl.lse, ws)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        step()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (steps * layers)


_FLUSH = {}


def flush_l2():
    import torch
    buf = _FLUSH.get("buf")
    if buf is None:
        buf = _FLUSH["buf"] = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")
    buf.fill_(float(len(_FLUSH)))


def cold_ms(wl: Workload, reps: int = 30, warmup: int = 5):
    """Kernel alone: median over `reps` single plain calls, each after an L2 flush (a write of
    2 x L2), bracketed by CUDA events on the launching stream (SURVEY §8(d) procedure)."""
    import torch
    l4, params, ws = make_l4(wl)
    st = torch.cuda.current_stream()
    ts = []
    for i in range(warmup + reps):
        flush_l2()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _call(l4, params, wl, i, ws)
        e1.record(st)
        e1.synchronize()
        if i >= warmup:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def plan_of(wl: Workload):
    l4, params, ws = make_l4(wl)
    q, k, v, ip, ix, kl = wl.sets[0]
    l4.decode_plan(params, kl, ip, wl.table.total_pages, ws)
    return l4.plan_info(ws)


def roofline_entry(wl: Workload, ms: float, peak: float, traffic_key: str = None):
    ach = wl.bytes_algo / (ms / 1e3) / 1e9
    ent = {"ms": round(ms, 5), "kv_gbs": round(wl.bytes_kv / (ms / 1e3) / 1e9, 1), "achieved": round(ach, 1),
           "frac": round(ach / peak, 4), "bytes_per_launch": wl.bytes_algo}
    if traffic_key:
        tr, src = measured_traffic(traffic_key)
        ent["traffic"] = tr
        if tr:
            ent["traffic_src"] = src
    return ent


# ----------------------------------------------------------------------------- e2e (CUDA graph)
def time_e2e(wl: Workload, steps: int):
    """The metric through the public API with HOST buffers.  Every step copies its inputs (q,
    kv_len, indptr, indices: packed in one pinned buffer, one H2D copy) to the device, runs
    l4_decode_attention and copies the fp32 output back (one D2H copy).  Copies run on their own
    streams and inputs / outputs / workspaces are double-buffered, so step i+1's H2D, step i's
    kernel and step i-1's D2H overlap.  The `steps`-step sequence (copies, events, kernels) is
    captured once in a CUDA graph and replayed: the timed region is one replay, from the first
    H2D to the last D2H; host_us_per_step is the host time of issuing that replay per step."""
    import torch
    from paper_2512_19179_b200 import l4
    params = l4.make_params(len(wl.lens), wl.shape.num_q_heads, wl.shape.num_kv_heads)
    ws = [l4.alloc_workspace(params, wl.table.total_pages) for _ in range(2)]
    q0, k, v, ip0, ix0, kl0 = wl.sets[0]
    parts = [q0, kl0, ip0, ix0]
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
        return [buf[o:o + t.numel() * t.element_size()].view(t.dtype).view(t.shape) for t, o in zip(parts, offs)]
    d_in = [views(d) for d in d_pack]
    d_out = [torch.empty(wl.out.shape, dtype=torch.float32, device="cuda") for _ in range(2)]
    d_lse = [torch.empty_like(wl.lse) for _ in range(2)]
    h_out = [torch.empty(wl.out.shape, dtype=torch.float32).pin_memory() for _ in range(2)]
    h2d = sum(t.numel() * t.element_size() for t in parts)
    d2h = h_out[0].numel() * h_out[0].element_size()
    s_main, s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    s_cmp = [torch.cuda.Stream(), torch.cuda.Stream()]
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_cmp = [torch.cuda.Event() for _ in range(2)]
    ev_out = [torch.cuda.Event() for _ in range(2)]

    def seq(n):
        cur = torch.cuda.current_stream()
        for s in (s_h2d, s_d2h, *s_cmp):
            s.wait_stream(cur)                     # fork from the capturing stream
        for i in range(n):
            b = i % 2
            if i >= 2:
                s_h2d.wait_event(ev_cmp[b])        # step i-2 finished reading these inputs
            with torch.cuda.stream(s_h2d):
                d_pack[b].copy_(h_pack, non_blocking=True)
            ev_in[b].record(s_h2d)
            s_cmp[b].wait_event(ev_in[b])
            if i >= 2:
                s_cmp[b].wait_event(ev_out[b])     # step i-2's output has been copied out
            q, kl, ip, ix = d_in[b]
            l4.attention_call(params, q, k, v, ip, ix, kl, wl.table.total_pages, d_out[b], d_lse[b], ws[b],
                              stream=s_cmp[b])
            ev_cmp[b].record(s_cmp[b])
            s_d2h.wait_event(ev_cmp[b])
            with torch.cuda.stream(s_d2h):
                h_out[b].copy_(d_out[b], non_blocking=True)
            ev_out[b].record(s_d2h)
        for s in (s_h2d, s_d2h, *s_cmp):
            cur.wait_stream(s)                     # join

    # eager warm-up (also sets the kernel attributes before capture), then capture
    with torch.cuda.stream(s_main):
        seq(4)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s_main):
        seq(steps)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_main)
    t0 = time.perf_counter()
    with torch.cuda.stream(s_main):
        graph.replay()
    host_s = time.perf_counter() - t0
    e1.record(s_main)
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    ok = torch.equal(d_out[(steps - 1) % 2].cpu(), h_out[(steps - 1) % 2])
    del graph
    return ms / steps, h2d, d2h, host_s * 1e6 / steps, ok


# ----------------------------------------------------------------------------- CPU baseline
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


def full_parity(names=("c1", "c2", "c3", "c4")):
    """Every output row of one plain GPU call against the FP64 oracle (all requests, all heads)
    at C1..C4, with the oracle's time (it gathers each request's pages from the device pools)."""
    import torch
    from oracle import attention as oa
    res = {}
    for name in names:
        spec = WORKLOADS[name]
        wl = Workload(name, spec["lens"](), spec["shape"], seed=7)
        l4, params, ws = make_l4(wl)
        _call(l4, params, wl, 0, ws)
        torch.cuda.synchronize()
        out, lse = wl.out.double().cpu().numpy(), wl.lse.double().cpu().numpy()
        q, k, v, _, _, _ = wl.sets[0]
        t0 = time.perf_counter()
        ro, rl = oa.paged_decode_attention(q, k, v, wl.table.indptr, wl.table.indices, wl.table.kv_len,
                                           wl.shape.num_kv_heads)
        dt = time.perf_counter() - t0
        res[name] = {"oracle_s": round(dt, 2), "max_abs_err_out": float(np.max(np.abs(out - ro))),
                     "max_abs_err_lse": float(np.max(np.abs(lse - rl))), "rows": int(out.shape[0] * out.shape[1]),
                     "oracle_gbs": round(wl.bytes_kv / dt / 1e9, 3)}
        del wl
        torch.cuda.empty_cache()
    return res


def partition_oracle_speed():
    """The partition oracle (pure Python, one core): M1 (C1: E = 4 over 40 requests) and the
    M5 / M6 inputs (10k ShareGPT-like requests, E = 4, 8, 16)."""
    from oracle import partition as op
    res = {}
    I, O = synth.requests_uniform(seed=0, n=40)
    t = time.perf_counter()
    op.plan_dp(I, O, 4, synth.roofline_qoe_d(), 7e11, 131072, mode=0)
    res["M1_E4_s"] = round(time.perf_counter() - t, 4)
    I, O = synth.requests_sharegpt_like(seed=1, n=10000)
    D = synth.roofline_qoe_d()
    for E in (4, 8, 16):
        t = time.perf_counter()
        op.plan_dp(I, O, E, D, 7e11, 131072, mode=0)
        res[f"M6_E{E}_s"] = round(time.perf_counter() - t, 3)
    return res


# ----------------------------------------------------------------------------- extra lines
def extra_lines(steps: int, warmup: int, peak: float):
    """C4, C2, the same C3 requests split into length bins, stage-shaped binned batches, short-
    request batches and the Fig. 2 analogue: steady (plain, rotating copies where they fit) and
    kernel-alone cold numbers, each as a roofline entry."""
    import torch
    res, roof = {}, {}

    def both(name, wl, traffic_key=None):
        ms = steady_ms(wl, steps, warmup)
        cold = cold_ms(wl)
        e = roofline_entry(wl, ms, peak, traffic_key)
        e["cold_ms"] = round(cold, 5)
        e["cold_frac"] = round(wl.bytes_algo / (cold / 1e3) / 1e9 / peak, 4)
        layers = 80 if wl.shape.num_q_heads == 64 else 32
        pl = per_layer_ms(wl, 2, 1, layers)  # 1 plan + `layers` runs per step (see per_layer_ms)
        e[f"per_layer_{layers}_ms"] = round(pl, 5)
        e[f"per_layer_{layers}_kv_gbs"] = round(wl.bytes_kv / (pl / 1e3) / 1e9, 1)
        roof[name] = e
        return e

    shape = synth.SHAPE_LLAMA3_8B
    for name in ("c4", "c2"):
        spec = WORKLOADS[name]
        wl = Workload(name, spec["lens"](), spec["shape"], copies=4 if name == "c2" else 2)
        both(name, wl, name)
        del wl
        torch.cuda.empty_cache()
    lens = synth.lengths_c3(0)
    edges = [0, 1024, 4096, 16384, 65536, 1 << 30]
    t_sum, b_sum, bins = 0.0, 0, []
    for lo, hi in zip(edges, edges[1:]):
        sel = lens[(lens >= lo) & (lens < hi)]
        if len(sel) == 0:
            continue
        w = Workload(f"c3[{lo},{hi})", sel, shape, copies=4)
        ms = steady_ms(w, steps, warmup)
        t_sum += ms
        b_sum += w.bytes_kv
        bins.append([lo, int(len(sel)), round(w.bytes_kv / (ms / 1e3) / 1e9, 1)])
        del w
    res["c3_same_requests_binned"] = {"kv_gbs": round(b_sum / (t_sum / 1e3) / 1e9, 1), "ms": round(t_sum, 4),
                                      "bins_lo_batch_gbs": bins}
    stage = []
    for lo, hi in zip(edges, edges[1:]):
        if not ((lens >= lo) & (lens < hi)).any():
            continue
        sl = _stage_lengths(lo, hi)
        w = Workload(f"stage[{lo}]", sl, shape, copies=2)
        e = both(f"stage{lo}", w, f"stage{lo}")
        stage.append([lo, int(sl[0]), len(sl), e["kv_gbs"]])
        del w
        torch.cuda.empty_cache()
    res["c3_stage_shaped_binned"] = stage
    short = []
    for sh, L in ((shape, 64), (shape, 200), (shape, 530), (synth.SHAPE_LLAMA3_70B, 64),
                  (synth.SHAPE_LLAMA3_70B, 200)):
        w = Workload(f"short{L}", np.full(1024, L, dtype=np.int64), sh, copies=4)
        key = f"short{'70b_' if sh.num_q_heads == 64 else ''}{L}"
        e = both(key, w, key)
        short.append([sh.name, L, round(e["ms"] * 1e3, 2), e["kv_gbs"], round(e["cold_ms"] * 1e3, 2)])
        del w
        torch.cuda.empty_cache()
    res["short_B1024_shape_L_us_gbs_coldus"] = short
    fig2 = []
    for s_len, l_len in ((1000, 50000), (200, 10000)):
        for kk in (1, 8, 32):
            mixed = synth.lengths_fig2(512, kk, s_len, l_len)
            homo = np.full(512, int(round(mixed.sum() / 512)), dtype=np.int64)
            t = []
            for lens_x in (mixed, homo):
                w = Workload("fig2", lens_x, shape, copies=2)
                t.append(steady_ms(w, steps, warmup))
                del w
            fig2.append([s_len, l_len, kk, round(t[0] / t[1], 3)])
    res["fig2_slowdown_short_long_k_ratio"] = fig2
    torch.cuda.empty_cache()
    return res, roof


def migration_bandwidth(reps: int = 10):
    """l4_copy_pages / l4_migrate of one request at the Llama-3-8B shape, all 32 layers: a
    2048-token request = 128 pages x 32 layers x (K, V) = 256 MiB, loopback on one GPU (HBM ->
    HBM), with torch's device copy of the same bytes as the loopback reference."""
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
    a_ = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    b_ = torch.empty_like(a_)
    t_torch = timed(lambda: b_.copy_(a_), reps)
    del k, v, k2, v2, a_, b_
    torch.cuda.empty_cache()
    return {"bytes": int(nbytes), "kernel_ms": round(t_kernel, 4),
            "kernel_gbs_moved": round(nbytes / (t_kernel / 1e3) / 1e9, 1),
            "torch_copy_same_bytes_ms": round(t_torch, 4)}


def partition_speed():
    """l4_partition (host C++) over 10,000 ShareGPT-like requests (lengths up to
    128K) at E = 4, 8, 16; the paper plans E = 16 in 0.06 s."""
    from paper_2512_19179_b200 import l4
    I, O = synth.requests_sharegpt_like(seed=1, n=10000)
    D = synth.roofline_qoe_d()
    res = {}
    for E in (4, 8, 16):
        t = time.perf_counter()
        l4.partition(I, O, E, D, 7e11, 131072, mode=0)
        res[f"E{E}_ms"] = round((time.perf_counter() - t) * 1e3, 3)
    return res


# ----------------------------------------------------------------------------- N = 1 line
def single_gpu_line(args, rank, world, local):
    import torch
    peak, peak_src = load_peaks()
    spec = WORKLOADS[args.workload]
    wl = Workload(args.workload, spec["lens"](), spec["shape"], seed=rank, copies=args.copies)
    steady_ms(wl, 2, args.warmup)                              # first-call setup, attributes
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    ms = steady_ms(wl, args.steps, args.warmup)                # the step: one plain launch
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t[0])
    early = steady_ms(wl, args.steps, args.warmup, early=True)
    eplan = steady_ms(wl, args.steps, args.warmup, early_plan=True)
    cold = cold_ms(wl)
    n_layers = 80 if wl.shape.num_q_heads == 64 else 32
    per_layer = per_layer_ms(wl, max(2, args.steps // 4), 1, n_layers) if len(wl.lens) <= 1024 else None
    info = plan_of(wl)
    e2e_steps = max(50, args.steps)
    e2e_ms, h2d, d2h, host_us, e2e_ok = time_e2e(wl, e2e_steps)
    value = world * wl.bytes_kv / (ms / 1e3) / 1e9
    head = roofline_entry(wl, ms, peak, args.workload)
    rceil, rceil_src = read_ceiling()
    extra, roof = {}, {}
    if rank == 0 and world == 1 and not args.no_extra:
        del wl.sets[1:]
        torch.cuda.empty_cache()
        extra, roof = extra_lines(max(5, args.steps // 2), 3, peak)
        extra["migration_loopback"] = migration_bandwidth()
        extra["partition_m6_ms"] = partition_speed()
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(args.workload, budget_s=12.0)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if not args.no_extra:
            cpu["partition_oracle_s"] = partition_oracle_speed()
            cpu["full_parity_vs_gpu"] = full_parity()
    if rank != 0:
        return None
    roof = {args.workload + "_cold": {"ms": round(cold, 5), "frac": round(wl.bytes_algo / (cold / 1e3) / 1e9 / peak, 4)},
            args.workload + "_early_inputs": {"ms": round(early, 5),
                                              "frac": round(wl.bytes_algo / (early / 1e3) / 1e9 / peak, 4)},
            args.workload + "_early_plan": {"ms": round(eplan, 5),
                                            "frac": round(wl.bytes_algo / (eplan / 1e3) / 1e9 / peak, 4)},
            **roof}
    if per_layer:
        roof[args.workload + f"_per_layer_{n_layers}"] = {
            "ms": round(per_layer, 5), "kv_gbs": round(wl.bytes_kv / (per_layer / 1e3) / 1e9, 1),
            "frac": round(wl.bytes_algo / (per_layer / 1e3) / 1e9 / peak, 4),
            "how": f"one decode step of a {n_layers}-layer model: 1 l4_decode_plan + {n_layers} l4_decode_run "
                   "(the work list is shared by every layer; each layer reads its own K/V, rotating copies); "
                   "device time per layer"}
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": args.workload, "desc": spec["desc"], "batch": int(len(wl.lens)),
                   "sum_kv_len": int(wl.lens.sum()), "kv_bytes_per_step": wl.bytes_kv,
                   "num_q_heads": wl.shape.num_q_heads, "num_kv_heads": wl.shape.num_kv_heads, "head_dim": 128,
                   "page_size": 16, "page_layout": "fragmented (seeded permutation)",
                   "l2": f"{args.copies} rotating copies of every input (q, K/V pools, page table; "
                         f"{wl.input_bytes / 1e9:.2f} GB each, >> 126 MB L2); kernel-alone lines flush L2",
                   "parallelism": f"replicas x{world}" if world > 1 else "single instance",
                   "plan": {"items": info.num_items, "chunk_pages": info.chunk_pages, "ctas": info.num_ctas},
                   "call": "l4_decode_attention, plain (no early-input overlap), back-to-back steps"},
        "tokens_per_s": round(world * len(wl.lens) / (ms / 1e3), 1),
        "tokens_per_s_depth_normalised": {
            "value": round(world * len(wl.lens) / (ms / 1e3) / (80 if wl.shape.num_q_heads == 64 else 32), 1),
            "layers": 80 if wl.shape.num_q_heads == 64 else 32,
            "note": "SURVEY 8(d): B / (n_layers x t_call), attention time only (Llama-3-8B 32 / -70B 80 layers)"},
        "pct_hbm_peak": round(100.0 * value / (world * peak), 2),
        "gpu_launches": args.steps * (1 if len(wl.lens) <= 1024 else 2),
        "clocks": clk,
        "roofline": {"bound": "hbm", "kernel": "decode_kernel<G, fused> (l4_decode_attention)",
                     "achieved": head["achieved"], "peak": peak, "unit": "GB/s", "frac": head["frac"],
                     "traffic": head.get("traffic"), "traffic_source": head.get("traffic_src"),
                     "peak_source": peak_src, "launch_ms": round(ms, 5), "bytes_per_launch": wl.bytes_algo,
                     "frac_of_nominal_8TBs": round(head["achieved"] / 8000.0, 4), "read_ceiling_gbs": rceil,
                     "frac_of_read_ceiling": round(head["achieved"] / rceil, 4) if rceil else None,
                     "read_ceiling_source": rceil_src, "configs": roof},
        "e2e": {"value": round(world * wl.bytes_kv / (e2e_ms / 1e3) / 1e9, 1), "unit": "GB/s",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "ms_per_step": round(e2e_ms, 5),
                "steps": e2e_steps, "host_us_per_step": round(host_us, 2), "output_copied_ok": bool(e2e_ok),
                "how": "CUDA graph of the per-step H2D copy, l4_decode_attention and D2H copy (double-buffered)"},
    }
    if cpu:
        line["cpu_baseline"] = cpu
    if extra:
        line["extra"] = extra
    # compact summary last: the driver keeps the tail of stdout
    line["summary"] = {k: v.get("kv_gbs", v.get("frac")) for k, v in roof.items()}
    line["summary"][args.workload] = round(wl.bytes_kv / (ms / 1e3) / 1e9, 1)
    return line


# ----------------------------------------------------------------------------- N > 1: pipeline
def measure_nvlink(rank, world, local, nbytes=1 << 30):
    """Rank 0: one large peer copy (torch device-to-device across GPUs = cudaMemcpyPeerAsync with
    peer access) and l4_copy_pages of 2048 scattered pages of the Llama-3-8B layout (32 KB K +
    32 KB V slices), device 0 -> device 1, both timed with CUDA events on the source device, then
    broadcast to every rank.  None if the ranks share one device (development harness) or the
    probe failed (the pipeline line then says so and assumes 7.7e11 B/s)."""
    import torch
    import torch.distributed as dist
    from paper_2512_19179_b200 import l4
    res = torch.zeros(3, dtype=torch.float64)
    if rank == 0 and world > 1 and torch.cuda.device_count() > 1 and os.environ.get("L4_FORCE_DEVICE") is None:
        try:
            peer = (local + 1) % torch.cuda.device_count()
            l4.enable_peer_access(peer)
            src = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{local}")
            dst = torch.empty(nbytes, dtype=torch.uint8, device=f"cuda:{peer}")

            def timed(fn, reps=10):
                for _ in range(2):
                    fn()
                torch.cuda.synchronize(local)
                torch.cuda.synchronize(peer)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(reps):
                    fn()
                e1.record()
                e1.synchronize()
                torch.cuda.synchronize(peer)
                return e0.elapsed_time(e1) / reps
            t_copy = timed(lambda: dst.copy_(src, non_blocking=True))
            pages, half = 2048, 2048 * 32768
            pool = lambda t, o: t[o:o + half].view(torch.bfloat16).view(pages, 8, 16, 128)
            sv = l4.kv_view(pool(src, 0), pool(src, half))
            dv = l4.kv_view(pool(dst, 0), pool(dst, half), device=peer)
            sp = np.random.default_rng(0).permutation(pages)
            dp = np.random.default_rng(1).permutation(pages)
            t_pages = timed(lambda: l4.copy_pages(sv, sp, dv, dp))
            res = torch.tensor([nbytes / (t_copy / 1e3), pages * 2 * sv.page_bytes / (t_pages / 1e3), float(peer)],
                               dtype=torch.float64)
            del src, dst
            torch.cuda.empty_cache()
        except Exception as e:  # noqa: BLE001 - the probe must not take the pipeline line down
            print(f"bench.py: NVLink probe failed: {e!r}"[:300], file=sys.stderr, flush=True)
            res = torch.zeros(3, dtype=torch.float64)
    cdev = torch.device("cuda", local) if dist.get_backend() == "nccl" else torch.device("cpu")
    res = res.to(cdev)
    dist.broadcast(res, 0)
    if float(res[0]) <= 0:
        return None
    return {"peer_copy_gbs": round(float(res[0]) / 1e9, 1), "l4_copy_pages_gbs": round(float(res[1]) / 1e9, 1),
            "bytes": nbytes, "pair": [0, int(res[2])],
            "how": "rank 0: 1 GiB device-to-device copy to the next GPU (peer access) and l4_copy_pages of 2048 "
                   "scattered pages (32 KB K + 32 KB V); CUDA events on the source device"}


def run_pipeline_arm(stages, steps, warmup, rank, world, device, per_rank=256, seed=0, shape=None, precopy_lead=0,
                     policy="least_loaded", rebalance_every=0, e2e=False, refine_every=0, qoe_d=None,
                     migrate_Bps=7.7e11):
    """C5: the length-aware pipeline on `world` GPUs.  Every step each rank runs the hot path
    (plan + split-KV kernel) on its resident batch, then the replicated control plane advances
    (tokens appended, handovers, retirements, arrivals, boundary refinement every
    `refine_every` steps) and KV pages of handed-over requests move between ranks on a copy
    stream (pipeline.DeviceOps).  With e2e=True every step also copies its batch's query rows in
    from pinned host memory and its attention output back to pinned host memory.
    Returns per-rank totals (device time measured with CUDA events on the compute stream)."""
    import torch
    import torch.distributed as dist
    from paper_2512_19179_b200 import l4, pipeline
    shape = shape or synth.SHAPE_LLAMA3_8B
    sim = pipeline.ClusterSim(stages, concurrency=world * per_rank, seed=seed, precopy_lead=precopy_lead,
                              policy=policy, rebalance_every=rebalance_every, refine_every=refine_every,
                              qoe_d=qoe_d, migrate_Bps=migrate_Bps)
    budget_pages = sim.token_budget // 16 * 5 // 4 + 2 * sim.batch_cap
    rt = pipeline.RankRuntime(sim, rank, budget_pages, shape, pipeline.DeviceOps(shape, device, seed + rank))
    if os.environ.get("L4_PIPE_TRANSPORT", "nccl") == "ipc" and world > 1:
        cpu_group = dist.new_group(backend="gloo") if dist.get_backend() != "gloo" else None
        rt.ops.setup_ipc(rt.pool, rank, world, cpu_group)
    cap = sim.batch_cap
    g = torch.Generator(device=device).manual_seed(seed + 100 + rank)
    q = torch.randn(cap, shape.num_q_heads, 128, device=device, generator=g).to(torch.bfloat16)
    out = torch.empty(cap, shape.num_q_heads, 128, dtype=torch.float32, device=device)
    lse = torch.empty(cap, shape.num_q_heads, dtype=torch.float32, device=device)
    if e2e:
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
    t_start = None
    hp = {} if os.environ.get("L4_HOST_PROFILE") else None   # development: host time per loop section

    def lap(key, t0):
        if hp is not None and t_start is not None:
            hp[key] = hp.get(key, 0.0) + time.perf_counter() - t0
        return time.perf_counter()
    for it in range(warmup + steps):
        timed = it >= warmup
        if it == warmup:
            rt.ops.drain()
            torch.cuda.synchronize()
            dist.barrier()
            rt.reset_stats()
            t_start = torch.cuda.Event(enable_timing=True)
            t_start.record(st)
            host_t0 = time.perf_counter()
        t0 = time.perf_counter()
        rt.ops.before_decode()                          # the step's decode waits for pages that landed
        kv_len, indptr = rt.device_batch()
        t0 = lap("device_batch", t0)
        B = int(kv_len.shape[0])
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        if B > 0:
            d_len, d_ptr = rt.ops.h2d.put(kv_len, indptr)
            t0 = lap("h2d_put", t0)
            params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads)
            qx, ox = q, out
            if e2e:
                bi = it % 2
                qx, ox = q_buf[bi], out_buf[bi]
                s_in.wait_event(ev_k[bi])
                if it == warmup:
                    s_in.wait_event(t_start)
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
        t0 = lap("attention_call", t0)
        rt.ops.after_decode(e1, e0)                      # pages freed this step wait for this decode
        ev = sim.step()
        t0 = lap("sim_step", t0)
        before = rt.stats["migrated_bytes"]
        rt.apply(ev, dist)
        t0 = lap("apply", t0)
        if timed:
            evs.append((e0, e1, B))
            tot["kv_bytes"] += int(4 * shape.num_kv_heads * 128 * int(kv_len.sum()))
            tot["launches"] = tot.get("launches", 0) + (1 if B > 0 else 0)
            tot["tokens"] += B
            tot["steps"] += 1
            tot["mig_bytes"] += rt.stats["migrated_bytes"] - before
            tot["mig_count"] += sum(1 for m in ev.migrations if m[1] == rank)
    host_ms = (time.perf_counter() - host_t0) * 1e3 / max(1, steps)  # enqueue time per step (host loop)
    rt.ops.drain()
    t_end = torch.cuda.Event(enable_timing=True)
    if e2e:
        st.wait_stream(s_out)
    t_end.record(st)
    torch.cuda.synchronize()
    for e0, e1, B in evs:
        dt = e0.elapsed_time(e1)
        tot["busy_ms"] += dt
        tot["lat_ms_x_req"] += dt * B
        tot["req_steps"] += B
    tot["elapsed_ms"] = t_start.elapsed_time(t_end)
    tot["host_ms_per_step"] = host_ms
    if hp is not None:
        print("host ms/step by section:", {k: round(v * 1e3 / max(1, steps), 4) for k, v in hp.items()},
              "h2d ring waits (ms, whole run):", round(rt.ops.h2d.wait_s * 1e3, 3), file=sys.stderr, flush=True)
    tot["launches"] = tot.get("launches", 0) + rt.stats["launches"]
    for k_ in ("precopy_pages", "stop_pages", "single_pages"):
        tot[k_] = rt.stats[k_]
    tot.update(rt.ops.transfer_stats())
    tot["fingerprint"] = sim.fingerprint()
    if hasattr(rt.ops, "close_ipc"):
        rt.ops.close_ipc()
    tot["stage_cv"] = sim.stage_cv()
    tot["stages"] = sim.current_stages()
    tot["refinements"] = sim.refinements
    return tot


def pipeline_line(args, world, rank, local):
    import torch
    import torch.distributed as dist
    from paper_2512_19179_b200 import pipeline
    device = torch.device("cuda", local)
    cdev = device if dist.get_backend() == "nccl" else torch.device("cpu")
    peak, peak_src = load_peaks()
    qoe_d, qoe_src = fitted_qoe_d()
    nvl = measure_nvlink(rank, world, local)
    bw = nvl["l4_copy_pages_gbs"] * 1e9 if nvl else 7.7e11
    stages, obj = pipeline.plan_stages(world, seed=0, qoe_d=qoe_d, bandwidth_Bps=bw)
    rr = [(0, stages[-1][1], world)]
    res = {}
    dist.barrier()
    ops = []   # warm up the NCCL P2P connections between every pair of ranks outside the timed region
    for peer in range(world):
        if peer != rank:
            ops.append(dist.P2POp(dist.isend, torch.ones(1, device=cdev), peer))
            ops.append(dist.P2POp(dist.irecv, torch.empty(1, device=cdev), peer))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    torch.cuda.synchronize()
    dist.barrier()
    # context: the same GPUs as independent replicas of the single-GPU C3 step (no pipeline, no
    # migration; what length-agnostic data parallelism over N instances moves), max over ranks
    rep = None
    try:
        spec = WORKLOADS["c3"]
        wlr = Workload("c3", spec["lens"](), spec["shape"], seed=rank, copies=2)
        steady_ms(wlr, 2, 3)
        dist.barrier()
        t_rep = torch.tensor([steady_ms(wlr, args.steps, args.warmup)], dtype=torch.float64, device=cdev)
        dist.all_reduce(t_rep, op=dist.ReduceOp.MAX)
        rep = {"kv_gbs": round(world * wlr.bytes_kv / (float(t_rep[0]) / 1e3) / 1e9, 1),
               "ms_per_step": round(float(t_rep[0]), 5),
               "note": "every rank runs the C3 single-GPU step on its own copy (plain calls); aggregate KV GB/s"}
        del wlr
        torch.cuda.empty_cache()
    except Exception as e:  # noqa: BLE001 - context only
        print(f"bench.py: replicas context failed: {e!r}"[:300], file=sys.stderr, flush=True)
    clocks = ClockSampler(local)
    clocks.start()
    clk = None
    arms = (("l4", stages, True, 0), ("l4_refined", stages, True, 10), ("round_robin", rr, False, 0),
            ("l4_e2e", stages, True, 0))
    for name, st, l4arm, refine in arms:
        # L4 arm (the value): l4_partition's stages, bid-ask receivers + intra-stage rebalancing
        # (P:391-399), live (two-round) migration with an 8-token pre-copy lead;
        # l4_refined: the same with boundary refinement every 10 steps (NEXT#2);
        # baseline: one length-agnostic stage, round-robin placement
        t = run_pipeline_arm(st, args.steps, args.warmup, rank, world, device,
                             precopy_lead=8 if l4arm else 0, policy="bidask" if l4arm else "round_robin",
                             rebalance_every=10 if l4arm else 0, e2e=name == "l4_e2e", refine_every=refine,
                             qoe_d=qoe_d, migrate_Bps=bw)
        if name == "l4":
            clk = clocks.stop()
        vec = torch.tensor([t["kv_bytes"], t["tokens"], t["mig_bytes"], t["mig_count"], t["req_steps"],
                            t["lat_ms_x_req"], t["launches"], t["precopy_pages"], t["stop_pages"],
                            t["single_pages"], t.get("h2d", 0), t.get("d2h", 0), t["busy_ms"],
                            t["stall_ms_sum"], t["stall_count"], t["copy_ms_sum"], t["copy_bytes"],
                            t["overlap_steps"]], dtype=torch.float64, device=cdev)
        dist.all_reduce(vec, op=dist.ReduceOp.SUM)
        tm = torch.tensor([t["elapsed_ms"], t["busy_ms"], t["stall_ms_max"], t["host_ms_per_step"]],
                          dtype=torch.float64, device=cdev)
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        fp = torch.tensor([t["fingerprint"] & 0x7FFFFFFF], dtype=torch.int64, device=cdev)
        fps = [torch.zeros_like(fp) for _ in range(world)]
        dist.all_gather(fps, fp)
        assert all(int(x) == int(fp) for x in fps), "replicated control plane diverged"
        elapsed = float(tm[0])
        res[name] = dict(kv_gbs=float(vec[0]) / (elapsed / 1e3) / 1e9, tokens_per_s=float(vec[1]) / (elapsed / 1e3),
                         elapsed_ms=elapsed, migrated_bytes=int(vec[2]), migrations=int(vec[3]),
                         mean_step_latency_ms=float(vec[5]) / max(1.0, float(vec[4])),
                         stage_cv=[round(x, 4) for x in t["stage_cv"]], launches=int(vec[6]),
                         precopy_pages=int(vec[7]), stop_round_pages=int(vec[8]), single_round_pages=int(vec[9]),
                         h2d_bytes=int(vec[10]), d2h_bytes=int(vec[11]), sum_busy_ms=float(vec[12]),
                         kv_bytes=float(vec[0]),
                         stall_ms_mean=float(vec[13]) / max(1.0, float(vec[14])), stall_ms_max=float(tm[2]),
                         copy_gbs=float(vec[16]) / max(1e-9, float(vec[15]) / 1e3) / 1e9 if vec[15] > 0 else None,
                         copy_overlapped_steps=int(vec[17]), host_ms_per_step_max=float(tm[3]),
                         stages=[list(x) for x in t["stages"]], refinements=t["refinements"])
    if rank != 0:
        return None
    l4r = res["l4"]
    line = {
        "metric": METRIC, "value": round(l4r["kv_gbs"], 1), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(l4r["elapsed_ms"] / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": "c5-pipeline", "desc": "BASELINE configs[4]: length-aware pipeline, "
                   f"{world} instances (1 GPU each), Llama-3-8B attention shape, ShareGPT-like closed loop, "
                   "256 resident requests per instance, 1.2M-token KV budget per instance",
                   "stages": stages, "partition_objective": obj, "qoe_d": list(qoe_d) if qoe_d else None,
                   "qoe_d_source": qoe_src, "migrate_bandwidth_Bps": bw,
                   "migrate_bandwidth_source": "measured in this run (l4_copy_pages over NVLink)" if nvl
                                               else "assumed 7.7e11 (ranks share one device)",
                   "parallelism": f"length-aware pipeline over {world} GPUs (l4_partition); KV migration "
                                  + ("one-sided over CUDA IPC (l4_copy_pages into peers' pools)"
                                     if os.environ.get("L4_PIPE_TRANSPORT", "nccl") == "ipc"
                                     else "over NCCL P2P (l4_pack_pages / l4_unpack_pages)")
                                  + " on a copy stream",
                   "l2": "inputs larger than L2; no flush"},
        "tokens_per_s": round(l4r["tokens_per_s"], 1),
        "pct_hbm_peak": round(100.0 * l4r["kv_gbs"] / (world * peak), 2),
        "gpu_launches": int(l4r["launches"]),
        "clocks": clk,
        "nvlink": nvl,
        "c3_replicas": rep,
        "pipeline": {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                     for k, v in res.items()},
    }
    ach = l4r["kv_bytes"] / (l4r["sum_busy_ms"] / 1e3) / 1e9 if l4r["sum_busy_ms"] > 0 else None
    line["roofline"] = {"bound": "hbm", "kernel": "decode_kernel<G, fused> (per-rank l4_decode_attention)",
                        "achieved": round(ach, 1) if ach else None, "peak": peak, "unit": "GB/s",
                        "frac": round(ach / peak, 4) if ach else None, "traffic": None, "peak_source": peak_src,
                        "note": "KV bytes only (q/out/ids not counted); per-GPU average"}
    e = res["l4_e2e"]
    line["e2e"] = {"value": round(e["kv_gbs"], 1), "unit": "GB/s",
                   "h2d_bytes_per_step": int(e["h2d_bytes"] / max(1, args.steps)),
                   "d2h_bytes_per_step": int(e["d2h_bytes"] / max(1, args.steps)),
                   "note": "the L4 arm again with every step's query rows copied in from pinned host memory and "
                           "its attention output copied back (bytes summed over ranks)"}
    line["summary"] = {k: [round(v["kv_gbs"], 1), round(v["tokens_per_s"], 1), round(v["mean_step_latency_ms"], 4),
                           v["migrations"]] for k, v in res.items()}
    line["summary"]["fields"] = ["kv_gbs", "tokens_per_s", "mean_step_latency_ms", "migrations"]
    return line


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


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    if rank != 0:
        return 0
    try:   # torchrun sets OMP_NUM_THREADS=1: the oracle gets every host core back
        import threadpoolctl
        threadpoolctl.threadpool_limits(limits=len(os.sched_getaffinity(0)))
    except Exception:
        pass
    name = args.workload
    spec = WORKLOADS[name]
    budget = args.sample_seconds or max(2.0, min(20.0, 60.0 / max(1, args.steps + args.warmup)))
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
    line = dict(impl="reference", metric=METRIC, value=round(v, 4), unit="GB/s", n_gpus=world,
                steps=args.steps, warmup=args.warmup, ms_per_step=round(ms_full, 3), higher_is_better=True,
                scaling="weak", vs_baseline=None, dtype="f64", data="synthetic",
                config=dict(workload=name, desc=spec["desc"], batch=len(spec["lens"]()),
                            kv_bytes_per_step=full_bytes),
                cpu_baseline=dict(value=round(v, 4), unit="GB/s", cores=samples["cores"], kind="oracle",
                                  sample=samples["sample"]),
                e2e=dict(value=round(v, 4), unit="GB/s", h2d_bytes_per_step=0, d2h_bytes_per_step=0))
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- main
def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def free_port() -> int:
    sk = socket.socket()
    sk.bind(("127.0.0.1", 0))
    port = sk.getsockname()[1]
    sk.close()
    return port


def spawn_command(argv, n: int, port: int):
    """`python bench.py --gpus N ...` without WORLD_SIZE: the same command under
    torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
            "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *argv]


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--workload", default="c3", choices=sorted(k for k in WORKLOADS if k != "c1"))
    ap.add_argument("--impl", default="l4", choices=["l4", "reference"])
    ap.add_argument("--copies", type=int, default=4, help="rotating input copies (L2 rotation)")
    ap.add_argument("--no-extra", action="store_true", help="skip the extra lines (C4, C2, binned, short, fig2)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU oracle baseline and full parity")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of the pipeline")
    ap.add_argument("--pipeline", action="store_true", help="run the C5 pipeline harness even at N = 1")
    ap.add_argument("--sample-seconds", type=float, default=0.0, help="reference arm: oracle seconds per step")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    world, rank, local = dist_env()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # the driver's form `python bench.py --gpus N`: become N ranks (one process per GPU)
        cmd = spawn_command(argv, args.gpus, free_port())
        return subprocess.call(cmd)
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        return run_reference(args, rank, world)

    import torch
    # development only: L4_FORCE_DEVICE pins every rank to one GPU and L4_PIPE_BACKEND=gloo swaps
    # NCCL for gloo (host-staged transport), so the N-rank harness runs on one B200
    local = int(os.environ.get("L4_FORCE_DEVICE", local))
    backend = os.environ.get("L4_PIPE_BACKEND", "nccl")
    torch.cuda.set_device(local)
    pipe = (world > 1 and not args.replicas) or args.pipeline
    if world > 1 or pipe:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")           # rank count visible in the NCCL init log
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        if world == 1:
            dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1,
                                    device_id=torch.device("cuda", local))
        elif backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if pipe:
        line = pipeline_line(args, world, rank, local)
    else:
        line = single_gpu_line(args, rank, world, local)
    if world > 1 or pipe:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
        if world > 1:
            time.sleep(1.0)  # let the other ranks' NCCL teardown log lines land before the JSON line
    if rank == 0 and line is not None:
        sys.stdout.flush()
        print(json.dumps(line), flush=True)  # the last line of stdout
    return 0


if __name__ == "__main__":
    sys.exit(main())
