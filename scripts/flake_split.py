"""Development: hunt the split-combine nondeterminism.

For a workload with split requests (default C4), repeat calls in one process and compare, bitwise,
every call's output AND the split partials left in the workspace against a first plain call:
  - a partial that differs => a split item was computed differently (ring / Q race);
  - equal partials but a different output => the combine itself;
  - NaN in the output (with --poison) => a combine read a partial before its split wrote it.
Usage: python scripts/flake_split.py [--wl c4|c3] [--iters N] [--poison] [--calls K] [--mode plain|early|both]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2512_19179_b200 import l4

ap = argparse.ArgumentParser()
ap.add_argument("--wl", default="c4")
ap.add_argument("--iters", type=int, default=40)
ap.add_argument("--calls", type=int, default=3)
ap.add_argument("--poison", action="store_true")
ap.add_argument("--mode", default="both")
ap.add_argument("--cks", action="store_true", help="debug variant built with -DL4_DEBUG_CKS: per-item data checksums")
ap.add_argument("--planrun", action="store_true", help="two-launch plan + run path instead of the single launch")
args = ap.parse_args()

if args.wl == "c4":
    shape, lens = synth.SHAPE_LLAMA3_70B, synth.lengths_c4(0)
elif args.wl == "c3":
    shape, lens = synth.SHAPE_LLAMA3_8B, synth.lengths_c3(0)
else:
    raise SystemExit("wl")
table = synth.make_page_table(lens, seed=0, spare_pages=64)
g = torch.Generator(device="cuda").manual_seed(0)
B = table.batch
q = torch.randn(B, shape.num_q_heads, 128, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
ip, ix, kl = (torch.from_numpy(x).cuda() for x in (table.indptr, table.indices, table.kv_len))


CKS_N = 16384 * 4


def cks_clear():
    if args.cks:
        torch.cuda.synchronize()
        assert l4.lib().l4_debug_cks(None, 0, 1) == 0


def cks_read():
    import ctypes
    buf = (ctypes.c_uint32 * CKS_N)()
    torch.cuda.synchronize()
    assert l4.lib().l4_debug_cks(buf, CKS_N, 0) == 0
    return np.frombuffer(buf, dtype=np.uint32).reshape(-1, 4).copy()


def call(params, ws, o, lz):
    cks_clear()
    if args.planrun:
        l4.decode_plan(params, kl, ip, table.total_pages, ws)
        l4.decode_run(params, q, k, v, ix, o, lz, ws)
    else:
        l4.attention_call(params, q, k, v, ip, ix, kl, table.total_pages, o, lz, ws)


p0 = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads)
ws0 = l4.alloc_workspace(p0, table.total_pages)
reg = l4.workspace_regions(p0, ws0.numel())
out = torch.empty(B, shape.num_q_heads, 128, device="cuda")
lse = torch.empty(B, shape.num_q_heads, device="cuda")
if args.poison:
    l4.poison_partials(p0, ws0)
call(p0, ws0, out, lse)
torch.cuda.synchronize()
ref_part = ws0[reg.partial_lse_offset:reg.end_offset].clone()
ref_cks = cks_read() if args.cks else None
print(f"{args.wl}: B={B} items_cap={reg.items_cap} partial bytes={ref_part.numel()}", flush=True)

modes = {"plain": [0], "early": [1], "both": [0, 1]}[args.mode]
fails = nan_fails = part_fails = 0
for it in range(args.iters):
    early = modes[it % len(modes)]
    params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads, flags=l4.L4_DECODE_EARLY_INPUTS if early else 0)
    ws = l4.alloc_workspace(params, table.total_pages)
    o2, l2 = torch.empty_like(out), torch.empty_like(lse)
    for c in range(args.calls):
        if args.poison:
            l4.poison_partials(params, ws)
        call(params, ws, o2, l2)
        if args.poison or args.cks or c == args.calls - 1:
            torch.cuda.synchronize()
            bad_out = not (torch.equal(o2, out) and torch.equal(l2, lse))
            part = ws[reg.partial_lse_offset:reg.end_offset]
            dp = part != ref_part
            n_part = int(dp.sum())
            has_nan = bool(torch.isnan(o2).any() or torch.isnan(l2).any())
            if bad_out or n_part:
                d = (o2 - out).abs().nan_to_num(float("inf"))
                rows = (d.amax(dim=2) > 0).nonzero()
                bh = sorted(set((int(r[0]), int(r[1]) // (shape.num_q_heads // shape.num_kv_heads)) for r in rows))
                first = int(dp.nonzero()[0]) if n_part else -1
                if n_part:
                    po = reg.partial_o_offset - reg.partial_lse_offset
                    slots = sorted(set(((dp.nonzero()[:, 0] - po) // (4 * 128 * (shape.num_q_heads // shape.num_kv_heads))).tolist()))
                    print(f"   partial slots differing (o region): {slots[:10]}", flush=True)
                if args.cks:
                    ck = cks_read()
                    bad = np.nonzero((ck != ref_cks).any(axis=1))[0]
                    for i in bad[:10]:
                        print(f"   item {i}: cks {ck[i].tolist()} ref {ref_cks[i].tolist()}", flush=True)
                print(f"iter {it} call {c} early={early}: out_bad={bad_out} nan={has_nan} max diff "
                      f"{float(d.max()):.3e} (b,kvh)={bh[:8]} n={len(bh)}; partial bytes differing={n_part} "
                      f"first at byte {first}", flush=True)
                fails += bad_out
                nan_fails += has_nan
                part_fails += n_part > 0
print(f"{os.environ.get('L4_LIB', 'libl4.so')} wl={args.wl} poison={args.poison} calls={args.calls}: "
      f"output mismatches {fails}, with NaN {nan_fails}, partial mismatches {part_fails} over {args.iters} iters")
