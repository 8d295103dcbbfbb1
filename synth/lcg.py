"""Counter-based input generator shared by the plain-C GPU client (tests/c/abi_gpu.c, which
re-implements it) and the golden-value writer (tests/golden/make_c1_decode_golden.py).  It holds
none of the method's arithmetic: it only draws bf16 values and a page permutation.

x_{n+1} = 6364136223846793005 * x_n + 1442695040888963407 (mod 2^64), x_0 = seed;
value(x) = (((x >> 33) mod 255) - 127) / 64, exactly representable in bf16 (7-bit magnitude).
"""
from __future__ import annotations

import numpy as np

A = 6364136223846793005
C = 1442695040888963407
M = (1 << 64) - 1


def values(seed: int, n: int) -> np.ndarray:
    """n float32 values (exact bf16) of the stream started at `seed`."""
    out = np.empty(n, dtype=np.float32)
    x = seed & M
    for i in range(n):
        x = (A * x + C) & M
        out[i] = (((x >> 33) % 255) - 127) / 64.0
    return out


def c1_problem():
    """BASELINE configs[0] on the LCG: Hq = 8, Hkv = 2, B = 4, L = {16, 64, 256, 1024}; pool of
    88 pages (3 spare), request pages laid out by indices[i] = (31 i + 7) mod 88; q, K, V from
    streams 1, 2, 3 in row-major order of [B, Hq, 128] and [88, Hkv, 16, 128]."""
    lens = np.array([16, 64, 256, 1024], dtype=np.int32)
    npg = (lens + 15) // 16
    indptr = np.zeros(5, dtype=np.int32)
    indptr[1:] = np.cumsum(npg)
    num_pages = int(indptr[-1]) + 3
    indices = ((31 * np.arange(indptr[-1]) + 7) % num_pages).astype(np.int32)
    q = values(1, 4 * 8 * 128).reshape(4, 8, 128)
    k = values(2, num_pages * 2 * 16 * 128).reshape(num_pages, 2, 16, 128)
    v = values(3, num_pages * 2 * 16 * 128).reshape(num_pages, 2, 16, 128)
    return lens, indptr, indices, num_pages, q, k, v
