"""Oracle: adaptive range refinement (§4.3) — TEST INFRASTRUCTURE ONLY.

  PAPER.md:369  "the instance collects the sequence lengths from both itself and its
                successors ... merges the successor sequence lengths as a union set, and
                divides the set evenly by the number of successors (using the same set
                division method in §4.2)"
  PAPER.md:372  "merges the instance's local sequence lengths and the average successor
                lengths into a single set ... sorts the requests ... as a list R"
  PAPER.md:374  b = argmin_{0 <= i < N} Q^{R[:i]} + Q^{R[i:]};  the boundary is the length R[b]
  PAPER.md:379  stability: initialised from the offline plan, exponential moving average,
                frozen when there are fewer than five requests

Readings (Z34-Z37):
  Z34 a tracked sequence is (I, L) with its true input length and current length L; Q^B of a
      list uses Eq. (1) with F4 = sum of current lengths (SPEC refiner decision).
  Z35 sort key for R and for the successor union: (L, I) ascending; the successor average is
      the canonical subset S[floor(k/2)::k] of the sorted union, k = number of successors.
  Z36 ties in the argmin go to the smallest i (first strict minimum).
  Z37 new boundary = alpha * R[b].L + (1 - alpha) * old, in float64, then clamped to
      [lo + 1, hi - 1] (strictly inside the two stages' outer bounds); with fewer than
      min_traffic merged requests (or none) the boundary is returned unchanged.
"""
from __future__ import annotations

import math

from .partition import batch_qoe, canonical_subset


class EmptyList(ValueError):
    pass


def _sorted(reqs):
    return sorted(((int(i), int(l)) for i, l in reqs), key=lambda r: (r[1], r[0]))


def average_successor_load(successor_sets):
    """Union of the successors' (I, L) sets, divided evenly by the number of successors."""
    k = len(successor_sets)
    if k == 0:
        return []
    union = _sorted([r for s in successor_sets for r in s])
    return canonical_subset(union, k)


def optimal_split(R, D):
    """b = argmin_{0 <= i < N} Q^{R[:i]} + Q^{R[i:]} over the sorted list R (smallest i on ties)."""
    N = len(R)
    if N == 0:
        raise EmptyList("empty list")
    best, b = math.inf, None
    for i in range(N):
        v = batch_qoe(R[:i], D) + batch_qoe(R[i:], D)
        if v < best:
            best, b = v, i
    return b


def refine(boundary: float, local, successor_sets, D, alpha: float, min_traffic: int, lo: int, hi: int):
    """One refinement of the boundary between a stage [lo, boundary) and its successor
    [boundary, hi).  Returns (new boundary, raw split length or None, split index or None)."""
    avg = average_successor_load(successor_sets)
    R = _sorted(list(local) + list(avg))
    if len(R) < min_traffic or len(R) == 0:      # P:379 freeze; nothing to split
        return float(boundary), None, None
    b = optimal_split(R, D)
    raw = R[b][1]
    nb = float(alpha) * float(raw) + (1.0 - float(alpha)) * float(boundary)
    nb = min(max(nb, float(lo + 1)), float(hi - 1))
    return nb, raw, b
