"""Oracle: paged GQA decode attention in FP64 — TEST INFRASTRUCTURE ONLY.

Follows the plain definition of one decode step's attention (the method —
split-KV plus a log-sum-exp combine — reaches exactly this result up to
rounding order, so the oracle is the definition written out):

  PAPER.md:94-97  "Each step reads all previously cached keys and values,
                   performing an attention operation with linear time
                   complexity, O(n), per request."
  PAPER.md:677    paged KV caches (vLLM).

Readings of points the paper leaves open (DESIGN.md §"Readings"):
  Z17 scale = 1/sqrt(D) unless given;  Z18 kv_head(h) = h // G;
  Z19 pools [num_pages, Hkv, P, D], CSR page table;  Z20 attend over
  tokens [0, L_b), no mask/window; token t lives at page
  indices[indptr[b] + t // P], slot t % P;  Z21 L_b = 0 -> out = 0,
  lse = -inf;  Z22 lse is the natural log.

Everything is computed in float64; bf16 inputs upcast exactly.
"""
from __future__ import annotations

import math

import numpy as np


def _to_f64(x) -> np.ndarray:
    """Exact upcast of a numpy array or a (CPU) torch tensor to float64."""
    if isinstance(x, np.ndarray):
        return x.astype(np.float64, copy=False)
    return x.detach().to("cpu").double().numpy()


def gather_request_kv(k_pages, v_pages, indptr, indices, kv_len, b: int, kv_head: int, page_size: int):
    """Dense K, V [L_b, D] of request b, kv head g, in logical token order (Z19/Z20)."""
    L = int(kv_len[b])
    if L == 0:
        return None, None
    s = int(indptr[b])
    n_pages = (L + page_size - 1) // page_size
    pages = np.asarray(indices[s:s + n_pages], dtype=np.int64)
    if isinstance(k_pages, np.ndarray):
        kb = k_pages[pages, kv_head]
        vb = v_pages[pages, kv_head]
    else:  # torch tensor (possibly on GPU): gather only this request's pages
        import torch
        idx = torch.as_tensor(pages, device=k_pages.device)
        kb = k_pages.index_select(0, idx)[:, kv_head]
        vb = v_pages.index_select(0, idx)[:, kv_head]
    K = _to_f64(kb).reshape(n_pages * page_size, -1)[:L]
    V = _to_f64(vb).reshape(n_pages * page_size, -1)[:L]
    return K, V


def attend_one(q: np.ndarray, K, V, scale: float):
    """out = sum_t softmax_t(scale * <q, k_t>) v_t and lse = ln sum_t exp(s_t).

    q: [D] float64; K, V: [L, D] float64 or None (L = 0).
    """
    D = q.shape[-1]
    if K is None or K.shape[0] == 0:
        return np.zeros(D, dtype=np.float64), -math.inf
    s = scale * (K @ q)                  # s_t = scale * sum_d q_d k_t,d
    m = float(np.max(s))                 # m = max_t s_t
    w = np.exp(s - m)                    # w_t = exp(s_t - m)
    Z = float(np.sum(w))                 # Z = sum_t w_t
    out = (w @ V) / Z                    # sum_t w_t v_t / Z
    lse = m + math.log(Z)                # lse = m + ln Z
    return out, lse


def paged_decode_attention(q, k_pages, v_pages, indptr, indices, kv_len,
                           num_kv_heads: int, page_size: int = 16, sm_scale: float | None = None,
                           requests=None, heads=None):
    """FP64 oracle for one decode iteration over a paged KV cache.

    q: [B, Hq, D] (numpy or torch, any float dtype); k_pages/v_pages:
    [num_pages, Hkv, P, D]; indptr [B+1], indices [indptr[B]], kv_len [B].
    ``requests``/``heads`` restrict the computation to a sample (for full-size
    parity on sampled outputs); entries outside the sample are NaN.
    Returns (out [B, Hq, D] float64, lse [B, Hq] float64).
    """
    qd = _to_f64(q)
    B, Hq, D = qd.shape
    G = Hq // num_kv_heads
    scale = (1.0 / math.sqrt(D)) if (sm_scale is None or sm_scale <= 0) else float(sm_scale)
    indptr = np.asarray(indptr, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    kv_len = np.asarray(kv_len, dtype=np.int64)
    out = np.full((B, Hq, D), np.nan, dtype=np.float64)
    lse = np.full((B, Hq), np.nan, dtype=np.float64)
    req_iter = range(B) if requests is None else requests
    for b in req_iter:
        head_iter = range(Hq) if heads is None else heads
        cache = {}
        for h in head_iter:
            g = h // G                                   # Z18: contiguous GQA groups
            if g not in cache:
                cache[g] = gather_request_kv(k_pages, v_pages, indptr, indices, kv_len, b, g, page_size)
            K, V = cache[g]
            out[b, h], lse[b, h] = attend_one(qd[b, h], K, V, scale)
    return out, lse


def lse_combine(parts):
    """Combine attention over disjoint token subsets: parts = [(out_s, lse_s)].

    With lse_s = ln Z_s and out_s = (sum_{t in s} w_t v_t) / Z_s, the whole-set
    result is out = sum_s (Z_s / Z) out_s with Z = sum_s Z_s, lse = ln Z
    (FlashDecoding aggregation).  Written with a max
    shift for range safety; empty parts (lse = -inf) contribute nothing.
    """
    lses = np.array([p[1] for p in parts], dtype=np.float64)
    if np.all(np.isneginf(lses)):
        return np.zeros_like(np.asarray(parts[0][0], dtype=np.float64)), -math.inf
    M = float(np.max(lses))
    w = np.exp(lses - M)
    Z = float(np.sum(w))
    out = sum(wi * np.asarray(p[0], dtype=np.float64) for wi, p in zip(w, parts)) / Z
    return out, M + math.log(Z)


def kv_bytes(kv_len, num_kv_heads: int, head_dim: int = 128, elem_bytes: int = 2) -> int:
    """Algorithmic KV bytes of one call: each valid K and V element read once
    (SURVEY.md §8(d) Roofline: 4*Hkv*D*sum(L) for bf16)."""
    return int(2 * num_kv_heads * head_dim * elem_bytes * int(np.sum(np.asarray(kv_len, dtype=np.int64))))
