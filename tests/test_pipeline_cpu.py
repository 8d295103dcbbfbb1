"""Multi-process CPU tests (gloo, world_size 2, 3 and 4) of the length-aware pipeline's host logic:
the replicated control plane agrees on every rank, the migration transport moves exactly the
migrating request's pages, page accounting is conserved, and the P2P exchange never deadlocks.
Device kernels are replaced by CPU mocks HERE (test-only); the product path uses libl4."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_19179_b200 import l4, pipeline


def test_assign_and_route():
    stages = [(0, 1024, 1), (1024, 4096, 2), (4096, 262144, 1)]
    assert pipeline.assign_ranks(stages) == [0, 1, 1, 2]
    sim = pipeline.ClusterSim(stages, concurrency=64, seed=1)
    assert sim.stage_of(0) == 0 and sim.stage_of(1023) == 0 and sim.stage_of(1024) == 1
    assert sim.stage_of(10 ** 9) == 2
    # every resident request sits on a rank of the stage covering its length or a later one
    for q in sim.reqs.values():
        assert sim.rank_stage[q.rank] == sim.stage_of(q.L)


def test_sim_placements_take_the_lowest_free_slot_and_skip_only_unplaceable_arrivals():
    """The control plane's fast paths change no decision: every placement takes the lowest inactive
    slot (the free-slot min-heap vs a scan of the active mask), and an arrival the pass skips
    through its capacity shortcut is one that no instance of its stage could take."""
    stages, _ = pipeline.plan_stages(4, seed=0, n_sample=2000)
    sim = pipeline.ClusterSim(stages, concurrency=4 * 256, seed=5, token_budget=300_000, policy="bidask",
                              rebalance_every=10, precopy_lead=8)
    orig_free, orig_ll = sim._free_slot, sim.least_loaded
    checked = {"slots": 0, "skips": 0}

    def free_slot():
        inactive = np.nonzero(~sim.active)[0]
        i = orig_free()
        if inactive.size:
            assert i == int(inactive[0])
            checked["slots"] += 1
        return i

    sim._free_slot = free_slot
    orig_place = sim._place

    def place(rid, I, O, L, initial=False, fail_cache=None):
        k = sim.stage_of(L)
        if fail_cache is not None and L + 1 >= fail_cache.get(k, 1 << 62):
            assert orig_ll(k, L + 1) is None     # the shortcut only skips what would fail anyway
            checked["skips"] += 1
        return orig_place(rid, I, O, L, initial=initial, fail_cache=fail_cache)

    sim._place = place
    for _ in range(300):
        sim.step()
    assert checked["slots"] > 100 and checked["skips"] > 0, checked


def test_sim_deterministic_and_conserving():
    stages, _ = pipeline.plan_stages(4, seed=0, n_sample=2000)
    a = pipeline.ClusterSim(stages, concurrency=256, seed=3)
    b = pipeline.ClusterSim(stages, concurrency=256, seed=3)
    n0 = len(a.reqs)
    for _ in range(300):
        ea, eb = a.step(), b.step()
        assert ea.migrations == eb.migrations and ea.retired == eb.retired and ea.admitted == eb.admitted
        # handovers go to the next stage, capped at 3 per sender
        for rid, src, dst, L, first in ea.migrations:
            assert a.rank_stage[dst] == a.rank_stage[src] + 1 or a.rank_stage[dst] > a.rank_stage[src]
        per_src = {}
        for _, src, _, _, _ in ea.migrations:
            per_src[src] = per_src.get(src, 0) + 1
        assert all(v <= 3 for v in per_src.values())
        # tokens bookkeeping equals the sum of resident lengths
        reqs = a.reqs
        for r in range(a.n_ranks):
            assert a.tokens[r] == sum(q.L for q in reqs.values() if q.rank == r)
    assert a.fingerprint() == b.fingerprint()
    assert len(a.reqs) + len(a.queue) >= n0 - 5


class MockOps:
    """CPU stand-in for DeviceOps (test only): pool pages are float32 tensors."""

    def __init__(self, page_elems=64):
        self.page_elems = page_elems

    def make_pool(self, num_pages):
        return dict(k=torch.zeros(num_pages, self.page_elems), v=torch.zeros(num_pages, self.page_elems),
                    alloc=l4.PagePool(num_pages))

    def alloc(self, pool, n):
        return pool["alloc"].alloc(n).tolist()

    def free(self, pool, pages):
        pool["alloc"].free(pages)

    def transfer(self, pool, sends, recvs, comm, any_transfer=None, joins=0, sent=0):
        ops, bufs, nbytes = [], [], 0
        for dst, pages in sends:
            idx = torch.tensor(pages, dtype=torch.long)
            st = torch.cat([pool["k"][idx], pool["v"][idx]], dim=1).contiguous()
            ops.append(dist.P2POp(dist.isend, st, dst))
            nbytes += st.numel() * 4
        for src, pages in recvs:
            st = torch.empty(len(pages), 2 * self.page_elems)
            ops.append(dist.P2POp(dist.irecv, st, src))
            bufs.append((pages, st))
            nbytes += st.numel() * 4
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for pages, st in bufs:
            idx = torch.tensor(pages, dtype=torch.long)
            pool["k"][idx] = st[:, :self.page_elems]
            pool["v"][idx] = st[:, self.page_elems:]
        return nbytes


def _worker(rank, world, port, stages, steps, out_q, lead=0, policy="least_loaded", rebalance_every=0,
            refine_every=0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sim = pipeline.ClusterSim(stages, concurrency=48 * world, seed=5, token_budget=400_000, batch_cap=256,
                                  precopy_lead=lead, policy=policy, rebalance_every=rebalance_every,
                                  refine_every=refine_every)
        ops = MockOps()
        rt = pipeline.RankRuntime(sim, rank, num_pages=400_000 // 16 * 2, shape=None, ops=ops)
        pool = rt.pool
        for rid, pages in rt.pages.items():          # tag every page with its owner
            pool["k"][torch.tensor(pages)] = float(rid)
            pool["v"][torch.tensor(pages)] = -float(rid)
        dist.barrier()
        checked = 0
        for _ in range(steps):
            before = {rid: len(p) for rid, p in rt.pages.items()}
            ev = sim.step()
            rt.apply(ev, dist)
            migrated_in = {m[0] for m in ev.migrations if m[2] == rank}
            for rid, pages in rt.pages.items():
                idx = torch.tensor(pages)
                if rid in migrated_in:               # every page arrived with its owner's tag
                    assert torch.all(pool["k"][idx] == float(rid)) and torch.all(pool["v"][idx] == -float(rid))
                    checked += 1
                else:
                    new = pages[before.get(rid, 0):]       # page lists only grow by appending
                    if new:
                        pool["k"][torch.tensor(new)] = float(rid)
                        pool["v"][torch.tensor(new)] = -float(rid)
            # page accounting: this rank owns exactly ceil(L/16) pages per resident request
            rids, Ls = sim.batch(rank)
            assert set(rids.tolist()) == set(rt.pages)
            for rid, L in zip(rids.tolist(), Ls.tolist()):
                assert len(rt.pages[rid]) == -(-L // 16)
            used = sum(len(p) for p in rt.pages.values()) + sum(len(p) for p in rt.incoming.values())
            assert pool["alloc"].num_free() == pool["alloc"].num_pages - used
        fps = [None] * world
        dist.all_gather_object(fps, (sim.fingerprint(), sim.rank_hi.tolist(), sim.refinements))
        out_q.put((rank, len(set(repr(f) for f in fps)) == 1, checked, dict(rt.stats, rank_hi=sim.rank_hi.tolist(),
                                                                           refinements=sim.refinements)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,lead,policy", [(2, 0, "least_loaded"), (3, 0, "least_loaded"), (2, 6, "least_loaded"),
                                               (3, 3, "least_loaded"), (4, 4, "bidask")])
def test_pipeline_gloo_migrations(world, lead, policy):
    """world 4 (bid-ask receivers, rebalancing checks every 10 steps, live migration): three
    stages, the middle one with two instances, so handovers go between four rank pairs
    (0->1, 0->2, 1->3, 2->3); the transport is the same for rebalancing moves."""
    if world == 4:
        stages = [(0, 1000, 1), (1000, 3000, 2), (3000, 262144, 1)]
    else:
        stages = [(0, 1500, 1), (1500, 262144, world - 1)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    reb = 10 if policy == "bidask" else 0
    procs = [ctx.Process(target=_worker, args=(r, world, port, stages, 120, q, lead, policy, reb))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res)
    total_checked = sum(c for _, _, c, _ in res)
    assert total_checked > 0                                # migrations actually happened and were verified
    outs = sum(s["migrations_out"] for *_, s in res)
    ins = sum(s["migrations_in"] for *_, s in res)
    assert outs == ins == total_checked
    stop = sum(s["stop_pages"] for *_, s in res)
    pre = sum(s["precopy_pages"] for *_, s in res)
    if lead > 0:   # live migration: most pages move in the pre-copy round, the stop round is small
        assert pre > 0 and stop > 0 and stop < pre
    else:
        assert pre == 0 and stop == 0


def test_detect_overload_examples():
    """strictly more than 25% above the stage mean."""
    assert not pipeline.detect_overload(100, [100, 100, 100, 100])
    assert pipeline.detect_overload(200, [100, 100, 100, 200])          # 200 > 1.25 * 125
    assert not pipeline.detect_overload(150, [100, 100, 150, 150])      # 150 < 1.25 * 125
    assert not pipeline.detect_overload(1.25 * 100, [100, 100, 100, 100], 1.25)   # boundary: not overloaded


def test_select_receiver_examples_and_properties():
    """lower-load half -> 3 earliest starts -> first reply, ties by id."""
    assert pipeline.select_receiver([(7, 5, 0.0, 0.0)]) == 7
    assert pipeline.select_receiver([(0, 10, 0, 0), (1, 20, 0, 0), (2, 30, 0, 0), (3, 40, 0, 0)]) == 0
    assert pipeline.select_receiver([]) is None
    rng = np.random.default_rng(0)
    for _ in range(2000):
        k = int(rng.integers(1, 12))
        bids = [(r, int(rng.integers(0, 50)), float(rng.integers(0, 5)), float(rng.random())) for r in range(k)]
        w = pipeline.select_receiver(bids)
        half = sorted(bids, key=lambda b: (b[1], b[0]))[: (k + 1) // 2]
        assert w in [b[0] for b in half]                                    # lower-load half
        early = sorted(half, key=lambda b: (b[2], b[0]))[:3]
        assert w in [b[0] for b in early]                                   # three earliest starts
        assert min(early, key=lambda b: (b[3], b[0]))[0] == w               # first reply


def test_bidask_balances_stages_fig16():
    """Fig. 16 (`fig:load-balancing`) analogue, 4 stages x 4 instances: per-stage CV of
    resident tokens with full bid-ask < bid-ask on handovers only < round-robin."""
    stages = [(0, 1024, 4), (1024, 4096, 4), (4096, 16384, 4), (16384, 262144, 4)]
    res = {}
    for name, pol, reb in (("rr", "round_robin", 0), ("inter", "bidask", 0), ("full", "bidask", 5)):
        cvs = []
        for seed in range(2):
            sim = pipeline.ClusterSim(stages, 16 * 16, seed=seed, policy=pol, rebalance_every=reb,
                                      token_budget=2_000_000)
            for s in range(500):
                ev = sim.step()
                for rid, src, dst, L, first in ev.migrations:       # rebalancing stays inside a stage
                    assert sim.rank_stage[dst] >= sim.rank_stage[src]
                if s >= 100 and s % 10 == 0:
                    cvs.append(np.mean(sim.stage_cv()))
        res[name] = float(np.mean(cvs))
    assert res["full"] < res["inter"] < res["rr"], res


def test_pipeline_gloo_refinement_moves_boundaries_and_ranks_agree():
    """NEXT#2 in the running pipeline: every 10 steps each instance refines its range
    boundary on the replicated state; over 120 steps the boundaries move, every rank computes the
    same boundaries, and handovers follow them with pages intact."""
    world = 3
    stages = [(0, 1500, 1), (1500, 262144, world - 1)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, stages, 120, q, 0, "least_loaded", 0, 10))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in res)                         # fingerprint + boundaries agree
    st = res[0][3]
    assert st["refinements"] == 12
    assert st["rank_hi"][0] != 1500.0                              # the first stage's boundary moved
    assert all(r[3]["rank_hi"] == st["rank_hi"] for r in res)
    assert sum(r[2] for r in res) > 0                              # migrations happened and were verified


def test_sim_refinement_equals_oracle_refine():
    """The boundary each instance gets from ClusterSim.refine is oracle/refine.py's result on that
    instance's (I, L) list and its successors' lists, with the stage's outer bounds (Z34-Z37)."""
    from oracle import refine as orf
    import synth
    stages = [(0, 1024, 2), (1024, 8192, 2), (8192, 262144, 1)]
    sim = pipeline.ClusterSim(stages, concurrency=300, seed=4, token_budget=10 ** 9)
    for _ in range(30):
        sim.step()
    per = [[] for _ in range(sim.n_ranks)]
    for i in np.nonzero(sim.active)[0]:
        per[int(sim.rank[i])].append((int(sim.I[i]), int(sim.L[i])))
    before = sim.rank_hi.copy()
    bounds = sim.bounds.copy()
    sim.refine()
    D = synth.roofline_qoe_d()
    for k in range(sim.last_stage):
        lo = 0 if k == 0 else int(np.floor(bounds[k - 1]))
        hi = int(sim.stage_hi[-1]) if k + 1 == sim.last_stage else int(np.ceil(bounds[k + 1]))
        succ = [per[r] for r in sim.stage_ranks[k + 1]]
        for r in sim.stage_ranks[k]:
            nb, _, _ = orf.refine(before[r], per[r], succ, D, 0.3, 5, lo, hi)
            assert sim.rank_hi[r] == nb
    for k in range(sim.last_stage):
        assert sim.bounds[k] == np.mean([sim.rank_hi[r] for r in sim.stage_ranks[k]])
    assert sim.rank_hi[-1] == before[-1]                            # the last stage has no upper boundary
