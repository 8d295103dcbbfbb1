"""Development: forensics of the wrong-V split partials.  Runs C4 with the -DL4_DEBUG_CKS
build until it catches calls whose per-item V checksum differs from a reference call, then finds
which page of the item was consumed with which data: for every page j of the item and every
candidate source (the V slice of page j + d of the same item, for |d| <= 16, or zeros, or one
64-column half of such a slice), it recomputes the item checksum the kernel would have produced
and reports the candidates that reproduce the observed value.

Checksum model (l4_decode.cu, L4_DEBUG_CKS): each consumer warp w XORs every 32-bit V fragment
register it loads (ldmatrix .trans: the low half holds an even token, the high half an odd token of
the same head_dim column), masked tokens contribute 0; the item value is XOR_w (cks_w * (2w + 1)),
and page j of a CTA-wide item is consumed by warp j % 4.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2512_19179_b200 import l4

ITERS = int(os.environ.get("ITERS", "3000"))
WANT = int(os.environ.get("WANT", "8"))
shape, lens = synth.SHAPE_LLAMA3_70B, synth.lengths_c4(0)
table = synth.make_page_table(lens, seed=0, spare_pages=64)
g = torch.Generator(device="cuda").manual_seed(0)
B = table.batch
q = torch.randn(B, shape.num_q_heads, 128, device="cuda", generator=g).to(torch.bfloat16)
k = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
v = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
ip, ix, kl = (torch.from_numpy(x).cuda() for x in (table.indptr, table.indices, table.kv_len))
N = 16384 * 4
M32 = np.uint64(0xFFFFFFFF)


def cks_read():
    buf = (ctypes.c_uint32 * N)()
    torch.cuda.synchronize()
    assert l4.lib().l4_debug_cks(buf, N, 0) == 0
    return np.frombuffer(buf, dtype=np.uint32).reshape(-1, 4).copy()


def call(params, ws, o, lz):
    torch.cuda.synchronize()
    assert l4.lib().l4_debug_cks(None, 0, 1) == 0
    l4.attention_call(params, q, k, v, ip, ix, kl, table.total_pages, o, lz, ws)


# the work list (same plan as the single launch)
p0 = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads)
ws0 = l4.alloc_workspace(p0, table.total_pages)
l4.decode_plan(p0, kl, ip, table.total_pages, ws0)
items = l4.plan_items(ws0)          # b, h, pbeg, pend, last_valid, part_base, nsplit, split
v_bits = v.view(torch.int16).cpu().numpy().view(np.uint16)     # [P, Hkv, 16, 128]


def page_cks(page, h, valid=16, half=None, rows=None, cols=None):
    x = v_bits[page, h].astype(np.uint32)
    if half is not None:
        x = x[:, half * 64:(half + 1) * 64]
    x = x.copy()
    x[valid:] = 0
    if rows is not None:
        x[~rows] = 0
    if cols is not None:
        x[:, ~cols] = 0
    lo = np.bitwise_xor.reduce(x[0::2].ravel()) if x[0::2].size else 0
    hi = np.bitwise_xor.reduce(x[1::2].ravel()) if x[1::2].size else 0
    return int(lo) | (int(hi) << 16)


def item_value(per_warp):
    out = 0
    for w in range(4):
        out ^= (per_warp[w] * (2 * w + 1)) & 0xFFFFFFFF
    return out


def analyse(i, observed, ref):
    b, h, pb, pe, lv = (int(x) for x in items[i][:5])
    pages = table.indices[pb:pe]
    np_ = len(pages)
    valid = [16] * np_
    valid[-1] = lv
    pc = [page_cks(int(pages[j]), h, valid[j]) for j in range(np_)]
    per_warp = [0, 0, 0, 0]
    for j in range(np_):
        per_warp[j % 4] ^= pc[j]
    model = item_value(per_warp)
    hits = []
    for j in range(np_):
        w = j % 4
        base = per_warp[w] ^ pc[j]
        cands = [("zeros", 0)]
        for d in range(-16, 17):
            jj = j + d
            if d == 0 or jj < 0 or jj >= np_:
                continue
            cands.append((f"page j{d:+d} full", page_cks(int(pages[jj]), h, valid[j])))
            for half in (0, 1):
                mixed = page_cks(int(pages[jj]), h, valid[j], half) ^ page_cks(int(pages[j]), h, valid[j], 1 - half)
                cands.append((f"page j{d:+d} half{half}", mixed))
            if abs(d) in (4, 8, 16):
                # partial overwrite: a contiguous block of tokens (rows) or of head_dim columns of
                # page j replaced by page j+d (the stage's next / previous use for d = +-8)
                for lo_ in range(16):
                    for hi_ in range(lo_ + 1, 17):
                        r = np.zeros(16, dtype=bool)
                        r[lo_:hi_] = True
                        mixed = page_cks(int(pages[jj]), h, valid[j], rows=r) ^ page_cks(int(pages[j]), h, valid[j], rows=~r)
                        cands.append((f"page j{d:+d} tokens[{lo_},{hi_})", mixed))
                for lo_ in range(0, 128, 8):
                    for hi_ in range(lo_ + 8, 129, 8):
                        c_ = np.zeros(128, dtype=bool)
                        c_[lo_:hi_] = True
                        mixed = page_cks(int(pages[jj]), h, valid[j], cols=c_) ^ page_cks(int(pages[j]), h, valid[j], cols=~c_)
                        cands.append((f"page j{d:+d} cols[{lo_},{hi_})", mixed))
        for name, c in cands:
            pw = list(per_warp)
            pw[w] = base ^ c
            if item_value(pw) == observed:
                hits.append((j, w, name))
    print(f"  item {i}: b {b} h {h} pages {np_} (model matches ref: {model == ref}); hypotheses reproducing the "
          f"observed checksum: {hits[:8]}", flush=True)


out, lse = torch.empty(B, shape.num_q_heads, 128, device="cuda"), torch.empty(B, shape.num_q_heads, device="cuda")
call(p0, ws0, out, lse)
ref = cks_read()
found = 0
for it in range(ITERS):
    params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads, flags=l4.L4_DECODE_EARLY_INPUTS)
    ws = l4.alloc_workspace(params, table.total_pages)
    o2, l2 = torch.empty_like(out), torch.empty_like(lse)
    for c in range(3):
        call(params, ws, o2, l2)
        ck = cks_read()
        bad = np.nonzero((ck != ref).any(axis=1))[0]
        for i in bad:
            print(f"iter {it} call {c}: item {i} cks {ck[i].tolist()} ref {ref[i].tolist()}", flush=True)
            analyse(int(i), int(ck[i][1]), int(ref[i][1]))
            found += 1
    if found >= WANT:
        break
print(f"found {found} bad items in {it + 1} iterations")
