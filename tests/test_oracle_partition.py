"""Pins for the partition oracle (oracle/partition.py): SPEC.md worked values,
the SURVEY A.2 hand example, exhaustive enumeration, objective decomposition
and invariants.
"""
import json
import os

import numpy as np
import pytest

import synth
from oracle import partition as op

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "partition_examples.json")))


@pytest.mark.parametrize("ex", GOLD["batch_features"], ids=lambda e: e["cite"][:40])
def test_batch_features_examples(ex):
    assert list(op.batch_features([tuple(r) for r in ex["reqs"]])) == ex["F"]


@pytest.mark.parametrize("ex", GOLD["request_qoe"], ids=lambda e: e["cite"][:40])
def test_request_qoe_examples(ex):
    assert op.request_qoe(ex["F"], ex["D"]) == ex["q"]


@pytest.mark.parametrize("ex", GOLD["batch_qoe"], ids=lambda e: e["cite"][:40])
def test_batch_qoe_examples(ex):
    assert op.batch_qoe([tuple(r) for r in ex["reqs"]], ex["D"]) == ex["QB"]


@pytest.mark.parametrize("ex", GOLD["canonical_subset"], ids=lambda e: e["cite"][:40])
def test_canonical_subset_examples(ex):
    assert op.canonical_subset(ex["set"], ex["m"]) == ex["subset"]


@pytest.mark.parametrize("ex", GOLD["cut_cost"], ids=lambda e: e["cite"][:40])
def test_cut_cost_examples(ex):
    reqs = [(i, i + o) for i, o in ex["reqs_IO"]]
    assert op.cut_cost(ex["cut"], reqs, ex["kv_bytes_per_token"], ex["bandwidth"]) == ex["c"]


@pytest.mark.parametrize("ex", GOLD["plans"], ids=lambda e: e["cite"][:50])
def test_plan_examples(ex):
    stages, obj = op.plan_dp(ex["I"], ex["O"], ex["E"], ex["D"], ex["bandwidth"], ex["kv_bytes_per_token"],
                             mode=ex["mode"])
    assert obj == ex["objective"]
    if "stages" in ex:
        assert [list(s) for s in stages] == ex["stages"]
    bp, bobj, _ = op.plan_bruteforce(ex["I"], ex["O"], ex["E"], ex["D"], ex["bandwidth"],
                                     ex["kv_bytes_per_token"], mode=ex["mode"])
    assert bobj == obj


def test_split_evenly_union_and_sizes():
    rng = np.random.default_rng(0)
    for _ in range(50):
        s = sorted(rng.integers(0, 100, size=rng.integers(0, 30)).tolist())
        m = int(rng.integers(1, 7))
        parts = op.split_evenly(s, m)
        assert sorted(sum(parts, [])) == s
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) <= 1
        assert op.canonical_subset(s, m) == parts[m // 2]


def test_default_edges():
    assert op.default_edges(14) == [0, 1, 2, 4, 8, 16]
    assert op.default_edges(16) == [0, 1, 2, 4, 8, 16, 32]          # Z10: top edge > 16
    assert op.default_edges(131072)[-1] == 262144
    assert op.default_edges(0) == [0, 1]


def test_validation():
    with pytest.raises(op.InvalidArgument):
        op.plan_dp([1], [1], 0, (0,) * 5, 1.0, 1)
    with pytest.raises(op.InvalidArgument):
        op.plan_dp([0], [1], 1, (0,) * 5, 1.0, 1)
    with pytest.raises(op.InvalidArgument):
        op.plan_dp([1], [1], 1, (0,) * 5, 0.0, 1)
    with pytest.raises(op.Infeasible):
        op.plan_dp([10], [10], 2, (0,) * 5, 1.0, 1, edges=[0, 4, 20])
    with pytest.raises(op.InvalidArgument):
        op.plan_dp([1], [1], 2, (0,) * 5, 1.0, 1, edges=[0, 4, 4, 8])


def test_empty_request_set():
    stages, obj = op.plan_dp([], [], 3, (1, 1, 1, 1, 1), 1.0, 1)
    assert obj == 0.0
    assert stages == [(0, 1, 3)]


def test_single_instance_is_batch_qoe():
    """E = 1: one stage over everything, objective = Q^B(all)."""
    I, O = synth.requests_uniform(seed=1, n=30)
    D = (0.3, 0.01, 1e-4, 1e-7, 2e-3)
    for mode in (0, 1):
        stages, obj = op.plan_dp(I, O, 1, D, 5e3, 7, mode=mode)
        reqs = [(int(i), int(i) + int(o)) for i, o in zip(I, O)]
        assert obj == op.batch_qoe(reqs, D)
        assert len(stages) == 1 and stages[0][2] == 1 and stages[0][0] == 0


def _random_workload(rng, small_edges):
    n = int(rng.integers(0, 41))
    if small_edges:
        I = rng.integers(1, 16, size=n)
        O = rng.integers(1, 16, size=n)
    else:
        I = rng.integers(1, 300, size=n)
        O = rng.integers(1, 300, size=n)
    D = tuple(float(x) if rng.random() < 0.8 else 0.0 for x in rng.random(5) * [1, 0.1, 0.01, 1e-4, 0.01])
    bw = float(rng.uniform(10, 1000))
    kvb = int(rng.integers(1, 9))
    return I.tolist(), O.tolist(), D, bw, kvb


def test_dp_equals_exhaustive_enumeration():
    """SPEC.md:684 acceptance shape: 50 random workloads, E in {2,3,4}, <= 6 buckets,
    <= 40 requests: exact (bitwise) objective match; identical plan when the optimum is unique."""
    rng = np.random.default_rng(2024)
    n_unique = 0
    for case in range(50):
        E = int(rng.choice([2, 3, 4]))
        I, O, D, bw, kvb = _random_workload(rng, small_edges=True)
        edges = [0, 2, 4, 8, 16, 32]       # 5 buckets, every final length (<= 30) covered
        for mode in (0, 1):
            stages, obj = op.plan_dp(I, O, E, D, bw, kvb, edges=edges, mode=mode)
            bplan, bobj, nbest = op.plan_bruteforce(I, O, E, D, bw, kvb, edges=edges, mode=mode)
            assert obj == bobj, (case, mode)
            assert sum(m for _, _, m in stages) == E
            if nbest == 1:
                n_unique += 1
                assert stages == bplan
    assert n_unique > 20


def test_dp_equals_exhaustive_default_edges():
    """Default power-of-two edges (E = 4 over 40 requests, I, O ~ U{1..512})."""
    for seed in range(3):
        I, O = synth.requests_uniform(seed=seed, n=40)
        D = (1e-3, 1e-4, 1e-6, 1e-9, 1e-5)
        for mode in (0, 1):
            stages, obj = op.plan_dp(I, O, 4, D, 1e4, 16, mode=mode)
            _, bobj, _ = op.plan_bruteforce(I, O, 4, D, 1e4, 16, mode=mode)
            assert obj == bobj


def test_objective_decomposition():
    """Reported objective = stage costs + interior cut costs, recomputed from scratch
    (the Fig. 4 `fig:topo-example` identity f_{3,8,6k} = 3Q+3Q+2Q+c_2k+c_4k)."""
    rng = np.random.default_rng(5)
    for _ in range(20):
        I, O, D, bw, kvb = _random_workload(rng, small_edges=False)
        E = int(rng.integers(1, 7))
        for mode in (0, 1):
            stages, obj = op.plan_dp(I, O, E, D, bw, kvb, mode=mode)
            edges = op.default_edges(max([i + o for i, o in zip(I, O)], default=0))
            # independent recomputation straight from Eq. (1) and the straddle rule
            reqs = [(i, i + o) for i, o in zip(I, O)]
            acc = 0.0
            for lo, hi, m in stages:
                S = sorted([(r, k) for k, r in enumerate(reqs) if lo <= r[1] < hi],
                           key=lambda x: (x[0][1], x[0][0], x[1]))
                S = [r for r, _ in S]
                if mode == 0:
                    sub = S[m // 2::m]
                    st = float(m) * (0.0 if not sub else float(len(sub)) * op.request_qoe(op.batch_features(sub), D))
                else:
                    st = None
                    for k in range(m):
                        sub = S[k::m]
                        qb = 0.0 if not sub else float(len(sub)) * op.request_qoe(op.batch_features(sub), D)
                        st = qb if st is None else st + qb
                c = 0.0 if lo == 0 else float(sum(lo for (i, lf) in reqs if i < lo < lf) * kvb) / bw
                acc = (acc + st) + c
            assert acc == obj
            assert op.plan_objective(stages, I, O, D, bw, kvb, mode=mode) == obj
            # contiguity and instance conservation
            assert stages[0][0] == 0 and stages[-1][1] == edges[-1]
            for a, b in zip(stages, stages[1:]):
                assert a[1] == b[0]
            assert sum(m for _, _, m in stages) == E


def test_fig4_decomposition_identity():
    """with cuts 2k/4k and 3+3+2 instances, the pipeline quality is
    3Q^{n_{0,2k}/3} + 3Q^{n_{2k,4k}/3} + 2Q^{n_{4k,6k}/2} + c_{2k} + c_{4k}."""
    I, O = synth.requests_uniform(seed=3, n=60, max_in=3000, max_out=2999)
    D = (1e-3, 1e-4, 0.0, 0.0, 1e-6)
    edges = [0, 2000, 4000, 6000]
    plan = [(0, 2000, 3), (2000, 4000, 3), (4000, 6000, 2)]
    obj = op.plan_objective(plan, I, O, D, 1e9, 131072, edges=edges, mode=0)
    reqs = [(int(i), int(i) + int(o)) for i, o in zip(I, O)]

    def Qsub(lo, hi, m):
        S = sorted([(r, k) for k, r in enumerate(reqs) if lo <= r[1] < hi], key=lambda x: (x[0][1], x[0][0], x[1]))
        return float(m) * op.batch_qoe([r for r, _ in S][m // 2::m], D)

    c = lambda cut: op.cut_cost(cut, reqs, 131072, 1e9)
    expect = ((((0.0 + Qsub(0, 2000, 3)) + 0.0 + Qsub(2000, 4000, 3)) + c(2000)) + Qsub(4000, 6000, 2)) + c(4000)
    assert abs(obj - expect) <= 1e-12 * abs(expect)


def test_mode1_monotone_in_instances():
    """Mode 1 with D >= 0: more instances never hurt (holds for mode 1 only, Z7)."""
    rng = np.random.default_rng(8)
    for _ in range(15):
        I, O, D, bw, kvb = _random_workload(rng, small_edges=False)
        prev = None
        for E in range(1, 6):
            _, obj = op.plan_dp(I, O, E, D, bw, kvb, mode=1)
            if prev is not None:
                assert obj <= prev
            prev = obj


def test_chain_not_better_than_exact():
    """plan_chain (1 instance per stage) is a restriction of the exact DP."""
    rng = np.random.default_rng(9)
    for _ in range(15):
        I, O, D, bw, kvb = _random_workload(rng, small_edges=False)
        E = int(rng.integers(1, 6))
        for mode in (0, 1):
            cst, cobj = op.plan_dp(I, O, E, D, bw, kvb, mode=mode, chain=True)
            _, obj = op.plan_dp(I, O, E, D, bw, kvb, mode=mode)
            assert cobj >= obj
            assert all(m == 1 for _, _, m in cst)


def test_modes_agree_at_scale():
    """with n >> m the literal footnote and the exact split choose the same plan."""
    I, O = synth.requests_sharegpt_like(seed=0, n=2000)
    D = synth.roofline_qoe_d()
    s0, _ = op.plan_dp(I, O, 4, D, 7e11, 131072, mode=0)
    s1, _ = op.plan_dp(I, O, 4, D, 7e11, 131072, mode=1)
    assert s0 == s1
    assert 2 <= len(s0) <= 4


def test_two_phase_never_beats_exact_and_merges_help():
    """Heuristic objective >= exact optimum; merging never increases the chain objective."""
    rng = np.random.default_rng(21)
    for _ in range(25):
        I, O, D, bw, kvb = _random_workload(rng, small_edges=False)
        E = int(rng.integers(1, 9))
        for mode in (0, 1):
            plan, obj = op.plan_two_phase(I, O, E, D, bw, kvb, mode=mode)
            _, exact = op.plan_dp(I, O, E, D, bw, kvb, mode=mode)
            assert obj >= exact
            assert sum(m for _, _, m in plan) == E
            edges = op.default_edges(max([i + o for i, o in zip(I, O)], default=0))
            J = len(edges) - 1
            if E <= J:
                _, chain = op.plan_dp(I, O, E, D, bw, kvb, mode=mode, chain=True)
                assert obj <= chain
            assert obj == op.plan_objective(plan, I, O, D, bw, kvb, mode=mode)


def test_two_phase_merges_when_cut_cost_dominates():
    """S:258 example: two stages whose migration cost at the cut dominates are merged into one."""
    I = [1, 2, 3, 40, 41, 42]
    O = [60, 60, 60, 2, 2, 2]                       # the short-input requests straddle every cut
    D = (0.0, 0.0, 0.0, 0.0, 1e-3)
    plan, obj = op.plan_two_phase(I, O, 2, D, 1.0, 10 ** 6)
    assert plan == [(0, 64, 2)]                     # one stage, no cut to pay
    # and with free migration the chain's two stages are kept
    # two well-separated groups and no straddlers: the chain's two stages are kept
    # (chain: 3*30 + 3*300 = 990 < merged 2 * 3 * (10 + 100 + 100) = 1260, D4 = 1)
    I2, O2 = [5, 5, 5, 50, 50, 50], [5, 5, 5, 50, 50, 50]
    plan2, obj2 = op.plan_two_phase(I2, O2, 2, (0, 0, 0, 0, 1.0), 1.0, 1)
    assert plan2 == [(0, 16, 1), (16, 128, 1)] and obj2 == 990.0
