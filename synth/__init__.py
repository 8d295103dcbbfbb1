"""Seeded synthetic input generators shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NONE of the method's arithmetic: it only draws lengths, page
tables, request (I, O) pairs and q/K/V values.  Neither the oracle
(``oracle/``) nor the CUDA path (``paper_2512_19179_b200``) imports the other;
both consume what this module produces.

The recipes are DESIGN.md §"Input recipe":

* C1 (M1): Hq=8, Hkv=2, D=128, P=16, B=4, L={16,64,256,1024}.
* C2 (M2): Llama-3-8B shape, Hq=32, Hkv=8, B=250, L=1024 for all.
* C3 (M3): Llama-3-8B shape, B=256, ShareGPT-like skew 100..128K: 248 short
  requests clip(round(exp(N(ln 1024, 1))), 100, 16383) and 8 long requests
  round(exp(U(ln 16384, ln 131072))), with short[0]=100 and long[-1]=131072.
  The paper prints no distribution parameters (Fig. 1 `fig:mixed-len`,
  PAPER.md:120-125 is an image); it states the shape only: "many short
  requests mixed with few but increasingly common long requests"
   and ">128K discarded".
* C4 (M4): Llama-3-70B shape, Hq=64, Hkv=8, B=32, L=round(U(32768, 131072))
  with L[0]=32768, L[-1]=131072.
* Partition workloads: (I, O) pairs, SURVEY.md §8(d) M1/M5/M6.

q/K/V values are i.i.d. N(0, 1) rounded to bf16 (torch CPU generator, seeded),
or drawn on the GPU with a seeded CUDA generator at full benchmark sizes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PAGE_SIZE = 16
HEAD_DIM = 128


@dataclass(frozen=True)
class AttnShape:
    name: str
    num_q_heads: int
    num_kv_heads: int
    head_dim: int = HEAD_DIM
    page_size: int = PAGE_SIZE

    @property
    def group(self) -> int:
        return self.num_q_heads // self.num_kv_heads


SHAPE_C1 = AttnShape("c1-8q2kv", 8, 2)
SHAPE_LLAMA3_8B = AttnShape("llama-3-8b", 32, 8)
SHAPE_LLAMA3_70B = AttnShape("llama-3-70b", 64, 8)


# ----------------------------------------------------------------------------
# Length distributions
# ----------------------------------------------------------------------------

def lengths_c1() -> np.ndarray:
    """BASELINE.json configs[0]: KV lengths {16, 64, 256, 1024}."""
    return np.array([16, 64, 256, 1024], dtype=np.int64)


def lengths_c2(batch: int = 250, length: int = 1024) -> np.ndarray:
    """BASELINE.json configs[1]: batch 250, uniform 1K contexts."""
    return np.full(batch, length, dtype=np.int64)


def lengths_c3(seed: int = 0, n_short: int = 248, n_long: int = 8) -> np.ndarray:
    """BASELINE.json configs[2]: batch 256 with ShareGPT-like skew 100..128K."""
    rng = np.random.default_rng(seed)
    short = np.clip(np.round(np.exp(rng.normal(math.log(1024.0), 1.0, n_short))), 100, 16383)
    long = np.round(np.exp(rng.uniform(math.log(16384.0), math.log(131072.0), n_long)))
    short = short.astype(np.int64)
    long = long.astype(np.int64)
    short[0] = 100
    long[-1] = 131072
    return np.concatenate([short, long])


def lengths_c3_production(seed: int = 0, n_short: int = 240, n_long: int = 16) -> np.ndarray:
    """SURVEY §8(d) M3 "production-like" variant of C3: batch 256, 16 long requests and a short
    median of 2048 (seed 0: sum L = 1,870,679)."""
    rng = np.random.default_rng(seed)
    short = np.clip(np.round(np.exp(rng.normal(math.log(2048.0), 1.0, n_short))), 100, 16383)
    long = np.round(np.exp(rng.uniform(math.log(16384.0), math.log(131072.0), n_long)))
    short = short.astype(np.int64)
    long = long.astype(np.int64)
    short[0] = 100
    long[-1] = 131072
    return np.concatenate([short, long])


def lengths_c4(seed: int = 0, batch: int = 32) -> np.ndarray:
    """BASELINE.json configs[3]: long-context batch 32 with lengths 32K..128K."""
    rng = np.random.default_rng(seed)
    lens = np.round(rng.uniform(32768.0, 131072.0, batch)).astype(np.int64)
    lens[0] = 32768
    lens[-1] = 131072
    return lens


def lengths_fig2(batch: int = 512, n_long: int = 8, short: int = 1000, long: int = 50000) -> np.ndarray:
    """Fig. 2 (`fig:interference`) analogue: k long + rest short."""
    lens = np.full(batch, short, dtype=np.int64)
    lens[:n_long] = long
    return lens


def random_lengths(rng: np.random.Generator, batch: int, lo: int, hi: int) -> np.ndarray:
    return rng.integers(lo, hi + 1, size=batch).astype(np.int64)


# ----------------------------------------------------------------------------
# Paged layout: CSR page table over a pool [num_pages, Hkv, P, D]
# ----------------------------------------------------------------------------

@dataclass
class PageTable:
    kv_len: np.ndarray          # int32 [B]
    indptr: np.ndarray          # int32 [B+1]
    indices: np.ndarray         # int32 [indptr[-1]]
    num_pages: int              # pool size (>= indptr[-1])

    @property
    def batch(self) -> int:
        return int(self.kv_len.shape[0])

    @property
    def total_pages(self) -> int:
        return int(self.indptr[-1])


def pages_for(length: int, page_size: int = PAGE_SIZE) -> int:
    return (int(length) + page_size - 1) // page_size


def make_page_table(kv_len, seed: int = 0, spare_pages: int = 0,
                    layout: str = "fragmented", page_size: int = PAGE_SIZE) -> PageTable:
    """CSR page table. ``fragmented`` = seeded random permutation of pool pages,
    ``contiguous`` = identity layout (SURVEY.md §8(d) "Page tables")."""
    kv_len = np.asarray(kv_len, dtype=np.int64)
    npages = np.array([pages_for(x, page_size) for x in kv_len], dtype=np.int64)
    indptr = np.zeros(len(kv_len) + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(npages)
    total = int(indptr[-1])
    num_pages = total + int(spare_pages)
    if layout == "fragmented":
        perm = np.random.default_rng(seed).permutation(num_pages)[:total]
    elif layout == "contiguous":
        perm = np.arange(total)
    else:
        raise ValueError(layout)
    return PageTable(kv_len=kv_len.astype(np.int32), indptr=indptr.astype(np.int32),
                     indices=perm.astype(np.int32), num_pages=max(num_pages, 1))


# ----------------------------------------------------------------------------
# q / K / V values (torch, bf16)
# ----------------------------------------------------------------------------

def make_qkv_cpu(shape: AttnShape, table: PageTable, seed: int = 0, q_scale: float = 1.0,
                 poison_unused: bool = True):
    """bf16 q [B,Hq,D], K/V pools [num_pages,Hkv,P,D] on CPU, N(0,1) rounded to bf16.

    With ``poison_unused`` every slot that no request may read (tails of last
    pages and pages outside the page table) is set to NaN, so an
    implementation that reads past kv_len is caught.
    """
    import torch

    g = torch.Generator().manual_seed(seed)
    B = table.batch
    q = (torch.randn(B, shape.num_q_heads, shape.head_dim, generator=g, dtype=torch.float32) * q_scale)
    k = torch.randn(table.num_pages, shape.num_kv_heads, shape.page_size, shape.head_dim,
                    generator=g, dtype=torch.float32)
    v = torch.randn(table.num_pages, shape.num_kv_heads, shape.page_size, shape.head_dim,
                    generator=g, dtype=torch.float32)
    q, k, v = q.to(torch.bfloat16), k.to(torch.bfloat16), v.to(torch.bfloat16)
    if poison_unused:
        poison_unread_slots(k, v, table, shape.page_size)
    return q, k, v


def valid_slot_mask(table: PageTable, page_size: int = PAGE_SIZE) -> np.ndarray:
    """bool [num_pages, P]: True where some request's token lives."""
    mask = np.zeros((table.num_pages, page_size), dtype=bool)
    for b in range(table.batch):
        L = int(table.kv_len[b])
        s, e = int(table.indptr[b]), int(table.indptr[b + 1])
        for j, p in enumerate(table.indices[s:e]):
            n = min(page_size, L - j * page_size)
            mask[p, :n] = True
    return mask


def poison_unread_slots(k, v, table: PageTable, page_size: int = PAGE_SIZE) -> None:
    import torch

    mask = torch.from_numpy(valid_slot_mask(table, page_size))  # [num_pages, P]
    bad = ~mask[:, None, :, None].expand_as(k)
    k.masked_fill_(bad, float("nan"))
    v.masked_fill_(bad, float("nan"))


# ----------------------------------------------------------------------------
# Partition workloads: (I, O) request pairs
# ----------------------------------------------------------------------------

def requests_uniform(seed: int = 0, n: int = 40, max_in: int = 512, max_out: int = 512):
    """I ~ U{1..512}, O ~ U{1..512}."""
    rng = np.random.default_rng(seed)
    I = rng.integers(1, max_in + 1, size=n).astype(np.int64)
    O = rng.integers(1, max_out + 1, size=n).astype(np.int64)
    return I, O


def requests_sharegpt_like(seed: int = 0, n: int = 10000, max_len: int = 131072):
    """I from the C3 generator family (31/32 short log-normal,
    1/32 long log-uniform), O = clip(round(exp(N(ln 256, 0.8))), 16, 4096), I+O <= max_len."""
    rng = np.random.default_rng(seed)
    is_long = rng.random(n) < (1.0 / 32.0)
    short = np.clip(np.round(np.exp(rng.normal(math.log(1024.0), 1.0, n))), 100, 16383)
    long = np.round(np.exp(rng.uniform(math.log(16384.0), math.log(120000.0), n)))
    I = np.where(is_long, long, short).astype(np.int64)
    O = np.clip(np.round(np.exp(rng.normal(math.log(256.0), 0.8, n))), 16, 4096).astype(np.int64)
    O = np.minimum(O, max_len - I)
    O = np.maximum(O, 1)
    return I, O


@dataclass
class QoeD:
    """D_0..D_4 of Eq. (1); inputs, never fitted here."""
    d: tuple = (0.0, 0.0, 0.0, 0.0, 1.0)
    extra: dict = field(default_factory=dict)


def roofline_qoe_d(kv_bytes_per_token_layer: float = 4096.0, layers: int = 32,
                   hbm_Bps: float = 6.5e12, step_overhead_s: float = 20e-6,
                   per_request_s: float = 0.2e-6) -> tuple:
    """a first-cut D from a B200 roofline (prefill not emulated)."""
    return (step_overhead_s, per_request_s, 0.0, 0.0, kv_bytes_per_token_layer * layers / hbm_Bps)
