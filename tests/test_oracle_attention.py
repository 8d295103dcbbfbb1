"""Pins for the FP64 attention oracle (oracle/attention.py) against things other
than itself: brute force, a library routine in float64, closed forms and
invariants.  The paper prints no attention values, so
there is no paper fixture: these pins are mathematical.
"""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import attention as oa


def _case(seed=0, lens=(16, 64, 37, 1), Hq=8, Hkv=2, q_scale=1.0, poison=True, layout="fragmented",
          spare=5):
    shape = synth.AttnShape("t", Hq, Hkv)
    table = synth.make_page_table(np.array(lens), seed=seed, spare_pages=spare, layout=layout)
    q, k, v = synth.make_qkv_cpu(shape, table, seed=seed, q_scale=q_scale, poison_unused=poison)
    return shape, table, q, k, v


def _run(shape, table, q, k, v, **kw):
    return oa.paged_decode_attention(q, k, v, table.indptr, table.indices, table.kv_len,
                                     shape.num_kv_heads, **kw)


def _brute_force(q, k, v, table, Hkv, scale):
    """Pure-Python triple loop over tokens with math.exp, no numpy reductions."""
    qd, kd, vd = q.double().numpy(), k.double().numpy(), v.double().numpy()
    B, Hq, D = qd.shape
    G = Hq // Hkv
    out = np.zeros((B, Hq, D))
    lse = np.zeros((B, Hq))
    for b in range(B):
        L = int(table.kv_len[b])
        for h in range(Hq):
            g = h // G
            scores = []
            for t in range(L):
                page = int(table.indices[int(table.indptr[b]) + t // 16])
                slot = t % 16
                acc = 0.0
                for d in range(D):
                    acc += float(qd[b, h, d]) * float(kd[page, g, slot, d])
                scores.append(scale * acc)
            if L == 0:
                lse[b, h] = -math.inf
                continue
            mx = max(scores)
            ws = [math.exp(s - mx) for s in scores]
            Z = sum(ws)
            for t in range(L):
                page = int(table.indices[int(table.indptr[b]) + t // 16])
                slot = t % 16
                for d in range(D):
                    out[b, h, d] += ws[t] * float(vd[page, g, slot, d])
            out[b, h] /= Z
            lse[b, h] = mx + math.log(Z)
    return out, lse


def test_bruteforce_tiny():
    shape, table, q, k, v = _case(lens=(3, 17, 0, 16), Hq=4, Hkv=2)
    out, lse = _run(shape, table, q, k, v)
    bo, bl = _brute_force(q, k, v, table, 2, 1.0 / math.sqrt(128))
    assert np.max(np.abs(out - bo)) < 1e-12
    finite = np.isfinite(bl)
    assert np.all(np.isneginf(lse[~finite]))
    assert np.max(np.abs(lse[finite] - bl[finite])) < 1e-12


def test_matches_torch_sdpa_float64():
    """Library special case: SDPA in float64 on the gathered dense K/V, KV repeated per group."""
    shape, table, q, k, v = _case(seed=3, lens=(1, 15, 16, 17, 300, 1024), Hq=8, Hkv=2)
    out, lse = _run(shape, table, q, k, v)
    G = shape.group
    for b in range(table.batch):
        L = int(table.kv_len[b])
        pages = table.indices[table.indptr[b]:table.indptr[b + 1]]
        K = k[torch.as_tensor(pages, dtype=torch.long)].double()      # [n, Hkv, 16, D]
        V = v[torch.as_tensor(pages, dtype=torch.long)].double()
        K = K.permute(1, 0, 2, 3).reshape(shape.num_kv_heads, -1, 128)[:, :L]
        V = V.permute(1, 0, 2, 3).reshape(shape.num_kv_heads, -1, 128)[:, :L]
        K = K.repeat_interleave(G, dim=0)
        V = V.repeat_interleave(G, dim=0)
        qb = q[b].double().unsqueeze(1)                                  # [Hq, 1, D]
        ref = torch.nn.functional.scaled_dot_product_attention(qb, K, V).squeeze(1)
        assert np.max(np.abs(out[b] - ref.numpy())) < 1e-12
        s = (qb @ K.transpose(1, 2)).squeeze(1) / math.sqrt(128)
        assert np.max(np.abs(lse[b] - torch.logsumexp(s, dim=-1).numpy())) < 1e-12


def test_closed_forms():
    # L = 1: out = v_0 exactly, lse = s_0.
    shape, table, q, k, v = _case(seed=1, lens=(1, 1, 1), Hq=4, Hkv=1)
    out, lse = _run(shape, table, q, k, v)
    for b in range(3):
        p = int(table.indices[table.indptr[b]])
        v0 = v[p, 0, 0].double().numpy()
        k0 = k[p, 0, 0].double().numpy()
        for h in range(4):
            assert np.array_equal(out[b, h], v0)
            s0 = float(np.dot(q[b, h].double().numpy(), k0)) / math.sqrt(128)
            assert abs(lse[b, h] - s0) < 1e-12
    # q = 0: uniform weights -> out = mean of V, lse = ln L.
    shape, table, q, k, v = _case(seed=2, lens=(5, 33, 200), Hq=4, Hkv=2)
    q.zero_()
    out, lse = _run(shape, table, q, k, v)
    for b in range(3):
        L = int(table.kv_len[b])
        for h in range(4):
            g = h // 2
            K, V = oa.gather_request_kv(k, v, table.indptr, table.indices, table.kv_len, b, g, 16)
            assert np.max(np.abs(out[b, h] - V.mean(axis=0))) < 1e-12
            assert abs(lse[b, h] - math.log(L)) < 1e-12
    # constant V = c: out = c for any q.
    shape, table, q, k, v = _case(seed=4, lens=(7, 100), Hq=4, Hkv=2, poison=False)
    v.fill_(0.75)
    out, _ = _run(shape, table, q, k, v)
    assert np.max(np.abs(out - 0.75)) < 1e-12
    # all keys equal: softmax uniform -> mean of V.
    shape, table, q, k, v = _case(seed=5, lens=(40,), Hq=2, Hkv=1, poison=False)
    k.copy_(k[0:1, :, 0:1, :].expand_as(k))
    out, _ = _run(shape, table, q, k, v)
    K, V = oa.gather_request_kv(k, v, table.indptr, table.indices, table.kv_len, 0, 0, 16)
    assert np.max(np.abs(out[0, 0] - V.mean(axis=0))) < 1e-12


def test_empty_request():
    shape, table, q, k, v = _case(lens=(0, 5, 0), Hq=4, Hkv=2)
    out, lse = _run(shape, table, q, k, v)
    assert np.all(out[0] == 0) and np.all(out[2] == 0)
    assert np.all(np.isneginf(lse[0])) and np.all(np.isneginf(lse[2]))
    assert np.all(np.isfinite(out[1]))


def test_page_layout_independence():
    """Permuting physical pages and rewriting indices leaves the result unchanged."""
    lens = (16, 31, 260, 5)
    shape, t1, q, k, v = _case(seed=7, lens=lens, layout="contiguous", spare=0, poison=False)
    out1, lse1 = _run(shape, t1, q, k, v)
    perm = np.random.default_rng(9).permutation(t1.num_pages)
    k2 = torch.empty_like(k)
    v2 = torch.empty_like(v)
    k2[torch.as_tensor(perm)] = k
    v2[torch.as_tensor(perm)] = v
    t2 = synth.PageTable(kv_len=t1.kv_len, indptr=t1.indptr,
                         indices=perm[t1.indices].astype(np.int32), num_pages=t1.num_pages)
    out2, lse2 = _run(shape, t2, q, k2, v2)
    assert np.array_equal(out1, out2) and np.array_equal(lse1, lse2)


def test_split_invariance():
    """Attention over any split of the tokens, LSE-combined, equals the unsplit result."""
    shape, table, q, k, v = _case(seed=11, lens=(300,), Hq=4, Hkv=1, poison=False)
    K, V = oa.gather_request_kv(k, v, table.indptr, table.indices, table.kv_len, 0, 0, 16)
    qv = q[0, 2].double().numpy()
    scale = 1 / math.sqrt(128)
    full = oa.attend_one(qv, K, V, scale)
    rng = np.random.default_rng(0)
    for _ in range(5):
        cuts = sorted(set(rng.integers(1, 300, size=4).tolist()))
        bounds = [0] + cuts + [300]
        parts = [oa.attend_one(qv, K[a:b], V[a:b], scale) for a, b in zip(bounds, bounds[1:])]
        parts.append(oa.attend_one(qv, K[:0], V[:0], scale))   # an empty split contributes nothing
        out, lse = oa.lse_combine(parts)
        assert np.max(np.abs(out - full[0])) < 1e-12
        assert abs(lse - full[1]) < 1e-12


def test_gqa_equals_mha_expansion():
    """Expanding each KV head to its G query heads (MHA) gives the same result."""
    shape, table, q, k, v = _case(seed=13, lens=(50, 17), Hq=8, Hkv=2, poison=False)
    out, lse = _run(shape, table, q, k, v)
    k_mha = k.repeat_interleave(4, dim=1)
    v_mha = v.repeat_interleave(4, dim=1)
    out2, lse2 = oa.paged_decode_attention(q, k_mha, v_mha, table.indptr, table.indices,
                                           table.kv_len, 8)
    assert np.array_equal(out, out2) and np.array_equal(lse, lse2)


def test_poisoned_tails_never_read():
    shape, table, q, k, v = _case(seed=17, lens=(1, 15, 17, 33), Hq=4, Hkv=2, poison=True)
    out, lse = _run(shape, table, q, k, v)
    assert np.all(np.isfinite(out)) and np.all(np.isfinite(lse))


def test_kv_bytes():
    assert oa.kv_bytes(synth.lengths_c2(), 8) == 1048576000
    assert oa.kv_bytes(synth.lengths_c3(0), 8) == 4 * 8 * 128 * 991974
