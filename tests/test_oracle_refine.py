"""Pins for the refinement oracle (oracle/refine.py): SPEC.md refiner examples,
an independent vectorised re-implementation of the argmin scan, EMA closed forms and the
low-traffic freeze."""
import math

import numpy as np
import pytest

from oracle import partition as op
from oracle import refine as orf


def test_average_successor_load_examples():
    # S:319 one successor [10, 20] -> itself; S:320 two successors, union [1..6] -> {2, 4, 6}
    assert orf.average_successor_load([[(1, 10), (1, 20)]]) == [(1, 10), (1, 20)]
    assert orf.average_successor_load([[(1, 1), (1, 3), (1, 5)], [(1, 2), (1, 4), (1, 6)]]) == [(1, 2), (1, 4), (1, 6)]
    assert orf.average_successor_load([]) == [] and orf.average_successor_load([[], []]) == []


def test_optimal_split_examples():
    assert orf.optimal_split([(3, 7)], (1, 1, 1, 1, 1)) == 0          # S:327 N = 1 -> b = 0
    with pytest.raises(orf.EmptyList):
        orf.optimal_split([], (1, 1, 1, 1, 1))
    # identical lengths, Q(S) = n * sum L (D4 = 1): i*(i*L) + (N-i)*((N-i)*L) is minimised
    # at i = N/2 (smallest index on ties)
    R = [(1, 10)] * 6
    assert orf.optimal_split(R, (0, 0, 0, 0, 1)) == 3


def _vectorised_split(R, D):
    """Independent implementation: prefix sums over the sorted list, all splits at once."""
    I = np.array([r[0] for r in R], dtype=np.int64)
    L = np.array([r[1] for r in R], dtype=np.int64)
    N = len(R)
    ci = np.concatenate([[0], np.cumsum(I)])
    ci2 = np.concatenate([[0], np.cumsum(I * I)])
    cl = np.concatenate([[0], np.cumsum(L)])
    vals = []
    for i in range(N):
        tot = 0.0
        for (n, si, si2, sl) in ((i, ci[i], ci2[i], cl[i]),
                                 (N - i, ci[N] - ci[i], ci2[N] - ci2[i], cl[N] - cl[i])):
            if n == 0:
                part = 0.0
            else:
                q = float(D[0]) * 1.0
                q = q + float(D[1]) * float(n)
                q = q + float(D[2]) * float(si)
                q = q + float(D[3]) * float(si2)
                q = q + float(D[4]) * float(sl)
                part = float(n) * q
            tot = part if tot == 0.0 and n == i else tot + part
        vals.append(tot)
    best = min(vals)
    return vals.index(best)


def test_optimal_split_matches_vectorised_scan():
    rng = np.random.default_rng(4)
    for _ in range(200):
        N = int(rng.integers(1, 40))
        R = sorted([(int(rng.integers(1, 500)), int(rng.integers(1, 5000))) for _ in range(N)],
                   key=lambda r: (r[1], r[0]))
        D = tuple(float(x) for x in rng.random(5) * np.array([1, 0.1, 1e-3, 1e-6, 1e-3]))
        assert orf.optimal_split(R, D) == _vectorised_split(R, D)


def test_refine_freeze_and_ema_degenerate_cases():
    local = [(1, 100), (1, 200)]
    succ = [[(1, 300), (1, 400)]]
    D = (0, 0, 0, 0, 1.0)
    # 4 requests < min_traffic 5 -> unchanged ("fewer than five requests")
    assert orf.refine(250.0, local, succ, D, 0.3, 5, 0, 10 ** 6) == (250.0, None, None)
    nb1, raw, b = orf.refine(250.0, local, succ, D, 1.0, 1, 0, 10 ** 6)   # alpha = 1 -> raw
    assert nb1 == float(raw)
    nb0, raw0, _ = orf.refine(250.0, local, succ, D, 0.0, 1, 0, 10 ** 6)  # alpha = 0 -> unchanged
    assert nb0 == 250.0
    nb, raw, _ = orf.refine(250.0, local, succ, D, 0.4, 1, 0, 10 ** 6)
    assert min(250.0, raw) <= nb <= max(250.0, raw)
    # clamping keeps the boundary strictly inside (lo, hi)
    nbc, _, _ = orf.refine(250.0, local, succ, D, 1.0, 1, 0, 150)
    assert nbc == 149.0


def test_refine_geometric_convergence():
    """with a fixed merged list, |b_t - raw| = (1 - alpha)^t |b_0 - raw|."""
    rng = np.random.default_rng(9)
    local = [(int(rng.integers(1, 50)), int(rng.integers(100, 2000))) for _ in range(20)]
    succ = [[(int(rng.integers(1, 50)), int(rng.integers(2000, 9000))) for _ in range(15)] for _ in range(3)]
    D = (1e-3, 1e-5, 0.0, 0.0, 1e-6)
    alpha, b0 = 0.3, 5000.0
    _, raw, _ = orf.refine(b0, local, succ, D, alpha, 5, 0, 10 ** 7)
    b = b0
    for t in range(1, 51):
        b, r, _ = orf.refine(b, local, succ, D, alpha, 5, 0, 10 ** 7)
        assert r == raw
        assert abs(abs(b - raw) - (1 - alpha) ** t * abs(b0 - raw)) <= 1e-9 * max(1.0, abs(b0 - raw))
