"""Oracle: L4 length-aware stage partition (§4.2) — TEST INFRASTRUCTURE ONLY.

Step by step in the paper's order and notation; every
reading of a silent/ambiguous point is listed in DESIGN.md §"Readings" (Z-ids).

  Eq. (1), PAPER.md:301-315   Q^B = n * sum_k D_k F_k, F = (1, n, sum I, sum I^2, sum L)
  PAPER.md:337-339            f_{s,e,l} = min_{e',l'} f_{s-1,e',l'} + (e-e') Q^{n_{l',l}/(e-e')} + c_{l'}
  PAPER.md:341                c_{l'} = transfer delay of fragments straddling the cut l'
  PAPER.md:342 (footnote)     set division S/n: sort, start at the n/2-th element, take every n-th
  PAPER.md:345                answer = min over s of f_{s,E,L}
  PAPER.md:357-358            cut candidates restricted to exponential buckets [1,2), [2,4), ...

Floating point (Z14): IEEE binary64 in a fixed operation order, no fused
multiply-add (Python floats never fuse), integer feature sums converted to
float once.  The C++ ``l4_partition`` must reproduce these bits exactly.
"""
from __future__ import annotations

import itertools
import math

INF = math.inf


# ---------------------------------------------------------------- validation

class InvalidArgument(ValueError):
    pass


class Infeasible(ValueError):
    pass


def validate(I, O, E: int, bandwidth: float):
    """Step 1: E >= 1, I_i >= 1, O_i >= 1, bandwidth > 0."""
    if E < 1:
        raise InvalidArgument("E must be >= 1")
    if not (bandwidth > 0):
        raise InvalidArgument("bandwidth must be > 0")
    if len(I) != len(O):
        raise InvalidArgument("I and O differ in length")
    for i, o in zip(I, O):
        if int(i) < 1 or int(o) < 1:
            raise InvalidArgument("input/output lengths must be >= 1")


# ---------------------------------------------------------------- Eq. (1)

def final_length(i: int, o: int) -> int:
    """Step 2, Z4: membership length of a request is its final length I + O."""
    return int(i) + int(o)


def batch_features(reqs):
    """F = (F0..F4) = (1, n, sum I, sum I^2, sum L) over reqs = [(I, L)] (Eq. (1)).

    Z8: L is the final length for planning.  Integer sums are exact."""
    n = len(reqs)
    return (1, n, sum(int(i) for i, _ in reqs), sum(int(i) * int(i) for i, _ in reqs),
            sum(int(l) for _, l in reqs))


def request_qoe(F, D) -> float:
    """Q_1 = sum_{k=0}^{4} D_k F_k, evaluated left to right: (((D0*F0 + D1*F1) + D2*F2) + D3*F3) + D4*F4."""
    q = float(D[0]) * float(F[0])
    q = q + float(D[1]) * float(F[1])
    q = q + float(D[2]) * float(F[2])
    q = q + float(D[3]) * float(F[3])
    q = q + float(D[4]) * float(F[4])
    return q


def batch_qoe(reqs, D) -> float:
    """Q^B = n * Q_1 (Eq. (1)); the empty batch costs 0."""
    if len(reqs) == 0:
        return 0.0
    F = batch_features(reqs)
    return float(F[1]) * request_qoe(F, D)


# ---------------------------------------------------------------- set division

def sort_key(req_with_index):
    """Z6: sort by (final length, input length, input index) ascending."""
    (i, lf), idx = req_with_index
    return (lf, i, idx)


def canonical_subset(sorted_reqs, m: int):
    """Footnote PAPER.md:342: start from the n/2-th element (Z5: 0-based floor(m/2)),
    then take every m-th.  e.g. [1..6] split 2 -> indices 1,3,5 -> {2,4,6}."""
    return sorted_reqs[m // 2::m]


def split_evenly(sorted_reqs, m: int):
    """All m strided subsets S[k::m] (mode 1, Z7)."""
    return [sorted_reqs[k::m] for k in range(m)]


def stage_cost(sorted_reqs, m: int, D, mode: int) -> float:
    """(e-e') * Q^{n_{l',l}/(e-e')}.

    mode 0 (paper-literal footnote): m * Q^B(S[floor(m/2)::m]).
    mode 1 (exact strided split):    sum_{k=0}^{m-1} Q^B(S[k::m]), summed in k order.
    """
    if mode == 0:
        return float(m) * batch_qoe(canonical_subset(sorted_reqs, m), D)
    if mode == 1:
        parts = split_evenly(sorted_reqs, m)
        acc = batch_qoe(parts[0], D)
        for k in range(1, m):
            acc = acc + batch_qoe(parts[k], D)
        return acc
    raise InvalidArgument("stage_cost_mode must be 0 or 1")


# ---------------------------------------------------------------- cut cost

def straddles(i: int, lf: int, cut: int) -> bool:
    """Z9: a request straddles cut l' iff I < l' < I + O (strict on both sides)."""
    return int(i) < cut < int(lf)


def cut_cost(cut: int, reqs, kv_bytes_per_token: int, bandwidth: float) -> float:
    """c_{l'}: every straddler moves the KV of l' tokens, in seconds."""
    tokens = sum(cut for (i, lf) in reqs if straddles(i, lf, cut))
    return float(tokens * int(kv_bytes_per_token)) / float(bandwidth)


# ---------------------------------------------------------------- buckets

def default_edges(max_lf: int):
    """Step 3, Z10: e_0 = 0, e_j = 2^(j-1) for j = 1..K+1,
    K = bit_length(max final length), so the top edge is > every final length."""
    K = int(max_lf).bit_length()
    return [0] + [1 << (j - 1) for j in range(1, K + 2)]


def check_edges(edges, max_lf: int):
    if len(edges) < 2 or edges[0] != 0:
        raise InvalidArgument("edges must start at 0 and have >= 2 entries")
    for a, b in zip(edges, edges[1:]):
        if not (b > a):
            raise InvalidArgument("edges must be strictly increasing")
    if edges[-1] <= max_lf:
        raise Infeasible("top edge must exceed the largest final length")


# ---------------------------------------------------------------- the DP

class _Problem:
    def __init__(self, I, O, E, D, bandwidth, kv_bytes_per_token, edges, mode):
        validate(I, O, E, bandwidth)
        self.E = int(E)
        self.D = tuple(float(x) for x in D)
        self.mode = int(mode)
        if self.mode not in (0, 1):
            raise InvalidArgument("stage_cost_mode must be 0 or 1")
        reqs = [(int(i), final_length(i, o)) for i, o in zip(I, O)]
        max_lf = max((lf for _, lf in reqs), default=0)
        self.edges = list(default_edges(max_lf) if edges is None else [int(x) for x in edges])
        check_edges(self.edges, max_lf)
        # Step 4: sort by (Lf, I, index).
        order = sorted(((r, k) for k, r in enumerate(reqs)), key=sort_key)
        self.sorted = [r for r, _ in order]
        self.reqs = reqs
        self.kvb = int(kv_bytes_per_token)
        self.bw = float(bandwidth)
        self._stage = {}
        self._cut = {}

    def slice(self, jp: int, j: int):
        """n_{l',l}: requests with e_{j'} <= Lf < e_j (Z3: half-open), in sorted order."""
        lo, hi = self.edges[jp], self.edges[j]
        return [r for r in self.sorted if lo <= r[1] < hi]

    def stage(self, jp: int, j: int, m: int) -> float:
        key = (jp, j, m)
        if key not in self._stage:
            self._stage[key] = stage_cost(self.slice(jp, j), m, self.D, self.mode)
        return self._stage[key]

    def cut(self, jp: int) -> float:
        """c at the stage's lower edge; the first stage (j' = 0) pays nothing."""
        if jp == 0:
            return 0.0
        if jp not in self._cut:
            self._cut[jp] = cut_cost(self.edges[jp], self.reqs, self.kvb, self.bw)
        return self._cut[jp]


def plan_dp(I, O, E, D, bandwidth, kv_bytes_per_token, edges=None, mode: int = 0,
            chain: bool = False):
    """Step 8-9: the exact DP over (s, e, j) with argmin recording.

    f[0][0][0] = 0, all other f[0] = +inf;  for s = 1..E, e = s..E, j = 1..J:
      f[s][e][j] = min over e' = s-1..e-1 (outer, ascending), j' = 0..j-1
                   (inner, ascending) of (f[s-1][e'][j'] + stage(j', j, e-e')) + c(j')
    keeping the first strict minimum (Z11: smaller e', then smaller j').
    Z1: e' <= e-1 so every stage has >= 1 instance.  Answer: min over s of
    f[s][E][J] with ties to the smaller s (Z12).  ``chain`` restricts every
    stage to one instance (the simplified DP of PAPER.md:360).
    Returns (stages [(lo, hi, instances)], objective).
    """
    p = _Problem(I, O, E, D, bandwidth, kv_bytes_per_token, edges, mode)
    E = p.E
    J = len(p.edges) - 1
    f = [[[INF] * (J + 1) for _ in range(E + 1)] for _ in range(E + 1)]
    arg = [[[None] * (J + 1) for _ in range(E + 1)] for _ in range(E + 1)]
    f[0][0][0] = 0.0
    for s in range(1, E + 1):
        for e in range(s, E + 1):
            for j in range(1, J + 1):
                best, best_arg = INF, None
                eps = [e - 1] if chain else range(s - 1, e)
                for ep in eps:
                    if ep < s - 1:
                        continue
                    for jp in range(0, j):
                        prev = f[s - 1][ep][jp]
                        if prev == INF:
                            continue
                        v = (prev + p.stage(jp, j, e - ep)) + p.cut(jp)
                        if v < best:
                            best, best_arg = v, (ep, jp)
                f[s][e][j] = best
                arg[s][e][j] = best_arg
    best_s, best = None, INF
    for s in range(1, E + 1):
        if f[s][E][J] < best:
            best_s, best = s, f[s][E][J]
    if best_s is None:
        raise Infeasible("no feasible plan")
    stages = []
    s, e, j = best_s, E, J
    while s > 0:
        ep, jp = arg[s][e][j]
        stages.append((p.edges[jp], p.edges[j], e - ep))
        s, e, j = s - 1, ep, jp
    stages.reverse()
    return stages, best


def plan_objective(stages, I, O, D, bandwidth, kv_bytes_per_token, edges=None, mode: int = 0) -> float:
    """Objective of a given plan, summed as the DP sums it: acc = (acc + stage_k) + c(lo_k)."""
    E = sum(m for _, _, m in stages)
    p = _Problem(I, O, E, D, bandwidth, kv_bytes_per_token, edges, mode)
    pos = {e: k for k, e in enumerate(p.edges)}
    acc = 0.0
    for lo, hi, m in stages:
        acc = (acc + p.stage(pos[lo], pos[hi], m)) + p.cut(pos[lo])
    return acc


def _compositions(E: int, s: int):
    """All ordered s-tuples of positive integers summing to E."""
    for cuts in itertools.combinations(range(1, E), s - 1):
        bounds = (0,) + cuts + (E,)
        yield tuple(bounds[k + 1] - bounds[k] for k in range(s))


def plan_bruteforce(I, O, E, D, bandwidth, kv_bytes_per_token, edges=None, mode: int = 0):
    """Step 10: exhaustive enumeration of every stage count s, every composition of
    E into s positive parts and every (s-1)-subset of interior edges; objective
    summed in the DP's order.  Returns (stages, objective, n_optimal_plans)."""
    p = _Problem(I, O, E, D, bandwidth, kv_bytes_per_token, edges, mode)
    E = p.E
    J = len(p.edges) - 1
    best, best_plan, n_best = INF, None, 0
    for s in range(1, E + 1):
        for comp in _compositions(E, s):
            for interior in itertools.combinations(range(1, J), s - 1):
                js = (0,) + interior + (J,)
                acc = 0.0
                for k in range(s):
                    acc = (acc + p.stage(js[k], js[k + 1], comp[k])) + p.cut(js[k])
                if acc < best:
                    best, n_best = acc, 1
                    best_plan = [(p.edges[js[k]], p.edges[js[k + 1]], comp[k]) for k in range(s)]
                elif acc == best:
                    n_best += 1
    return best_plan, best, n_best


# ---------------------------------------------------------------- two-phase heuristic

def plan_two_phase(I, O, E, D, bandwidth, kv_bytes_per_token, edges=None, mode: int = 0):
    """"We first run a simplified DP that assigns exactly one instance per stage,
    yielding an initial E-stage pipeline ... We then iteratively merge adjacent stages to
    reduce total latency. For each pair, we define a merge gain — the reduction in latency
    from unifying their instance and sequence range — and greedily merge the pair with the
    highest positive gain ... until no further improvement is possible."

    Readings (Z31-Z33):
      Z31 phase 1 is the chain DP with E1 = min(E, J) single-instance stages (J = number of
          buckets); if E > J, each remaining instance goes to the stage whose cost drops most
          when it gains one instance (ties: leftmost stage).
      Z32 merge gain of adjacent stages A, B = ((cost(A) + cost(B)) + c(B.lo)) - cost(A u B),
          A u B covering [A.lo, B.hi) with m_A + m_B instances; the pair with the largest
          strictly positive gain is merged first (ties: leftmost pair).
      Z33 the reported objective is recomputed from the final plan in the DP's summation order.
    This is the obviously-correct naive O(E^2) scan; the library uses a max-heap.
    """
    p = _Problem(I, O, E, D, bandwidth, kv_bytes_per_token, edges, mode)
    J = len(p.edges) - 1
    E1 = min(p.E, J)
    stages, _ = plan_dp(I, O, E1, D, bandwidth, kv_bytes_per_token, edges=p.edges, mode=mode, chain=True)
    pos = {e: k for k, e in enumerate(p.edges)}
    st = [[pos[lo], pos[hi], m] for lo, hi, m in stages]
    for _ in range(p.E - E1):                       # Z31: place the remaining instances
        best, best_k = None, None
        for k, (a, b, m) in enumerate(st):
            g = p.stage(a, b, m) - p.stage(a, b, m + 1)
            if best is None or g > best:
                best, best_k = g, k
        st[best_k][2] += 1
    while len(st) > 1:                              # Z32: greedy adjacent merges
        best, best_k = 0.0, None
        for k in range(len(st) - 1):
            (a, b, m1), (b2, c, m2) = st[k], st[k + 1]
            before = (p.stage(a, b, m1) + p.stage(b2, c, m2)) + p.cut(b2)
            gain = before - p.stage(a, c, m1 + m2)
            if gain > best:
                best, best_k = gain, k
        if best_k is None:
            break
        (a, _, m1), (_, c, m2) = st[best_k], st[best_k + 1]
        st[best_k:best_k + 2] = [[a, c, m1 + m2]]
    plan = [(p.edges[a], p.edges[b], m) for a, b, m in st]
    return plan, plan_objective(plan, I, O, D, bandwidth, kv_bytes_per_token, edges=p.edges, mode=mode)
