"""GPU test of the pipeline data path on one device: two RankRuntimes (two "instances") share
cuda:0 and exchange KV pages through an in-process loopback transport that mimics
torch.distributed's batched P2P API.  Checks: migrated pages are byte-identical to the
source pages (l4_pack_pages / l4_unpack_pages), and decode attention on the runtime's page
tables matches the FP64 oracle before and after migrations."""
import numpy as np
import pytest
import torch

import synth
from oracle import attention as oa
from paper_2512_19179_b200 import l4, pipeline

pytestmark = pytest.mark.gpu


class _Hub:
    """In-process stand-in for torch.distributed P2P between ranks of one process.
    Valid for forward-only pipelines processed in rank order (sends before receives)."""

    class P2POp:
        def __init__(self, op, tensor, peer):
            self.op, self.tensor, self.peer = op, tensor, peer

    def __init__(self):
        self.mail = {}
        self.me = 0

    @staticmethod
    def get_backend():  # device tensors move as with NCCL (no host staging)
        return "nccl"

    def isend(self):  # markers only
        pass

    def irecv(self):
        pass

    def batch_isend_irecv(self, ops):
        for o in ops:
            if o.op == self.isend:
                self.mail.setdefault((self.me, o.peer), []).append(o.tensor.clone())
        for o in ops:
            if o.op == self.irecv:
                o.tensor.copy_(self.mail[(o.peer, self.me)].pop(0))

        class _W:
            def wait(self):
                pass
        return [_W() for _ in ops]


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _attention_check(rt, shape, q):
    kv_len, indptr, indices = rt.tables()
    B = len(kv_len)
    if B == 0:
        return 0
    out, lse = l4.decode_attention(q[:B], rt.pool["k"], rt.pool["v"], torch.from_numpy(indptr).cuda(),
                                   torch.from_numpy(indices).cuda(), torch.from_numpy(kv_len).cuda())
    torch.cuda.synchronize()
    sample = sorted(set([0, B - 1, B // 2]))
    ro, rl = oa.paged_decode_attention(q[:B], rt.pool["k"], rt.pool["v"], indptr, indices, kv_len,
                                       shape.num_kv_heads, requests=sample)
    o = out.double().cpu().numpy()
    err = max(np.max(np.abs(o[b] - ro[b])) for b in sample)
    assert err <= 2e-3, err
    return B


@pytest.mark.parametrize("lead", [0, 4])
def test_two_instances_loopback_migration(lead):
    shape = synth.AttnShape("t", 8, 2)
    # put the stage boundary just above the median resident length so handovers happen soon
    probe = pipeline.ClusterSim([(0, 1 << 21, 2)], concurrency=40, seed=2, token_budget=10 ** 9, batch_cap=128)
    Ls = sorted(q.L for q in probe.reqs.values())
    cut = Ls[len(Ls) // 2] + 8
    stages = [(0, cut, 1), (cut, 1 << 21, 1)]
    sim = pipeline.ClusterSim(stages, concurrency=40, seed=2, token_budget=10 ** 9, batch_cap=128, precopy_lead=lead)
    ops = pipeline.DeviceOps(shape, "cuda", seed=1)
    rts = [pipeline.RankRuntime(sim, r, 60000, shape, ops) for r in range(2)]
    hub = _Hub()
    q = torch.randn(128, shape.num_q_heads, 128, device="cuda").to(torch.bfloat16)
    n_mig = 0
    for step in range(40):
        if step % 10 == 0:
            for rt in rts:
                _attention_check(rt, shape, q)
        ev = sim.step()
        # the token each request produced this step is appended on its current owner before any
        # handover: write it into the owner's partial page (a stale pre-copied page then shows)
        for rt in rts:
            for rid, pages in rt.pages.items():
                L = sim.reqs[rid].L if rid in sim.reqs else None
                if L is None:
                    continue
                pidx, slot = (L - 1) // 16, (L - 1) % 16
                if pidx < len(pages):
                    val = float((rid * 7 + L) % 251) / 8.0
                    rt.pool["k"][pages[pidx], :, slot, :] = val
                    rt.pool["v"][pages[pidx], :, slot, :] = -val
        # snapshot the source pages of migrating requests (after this step's growth allocation
        # the source packs exactly these pages plus possibly one new page)
        snaps = {}
        for rid, src, dst, L, first in ev.migrations:
            pages = list(rts[src].pages[rid])
            snaps[rid] = (rts[src].pool["k"][torch.tensor(pages, device="cuda")].clone(),
                          rts[src].pool["v"][torch.tensor(pages, device="cuda")].clone(), len(pages))
        for r in range(2):
            hub.me = r
            rts[r].apply(ev, hub)
        torch.cuda.synchronize()
        for rid, src, dst, L, first in ev.migrations:
            k0, v0, n0 = snaps[rid]
            pages = rts[dst].pages[rid]
            assert len(pages) == -(-L // 16)
            idx = torch.tensor(pages[:n0], device="cuda")
            assert torch.equal(rts[dst].pool["k"][idx], k0) and torch.equal(rts[dst].pool["v"][idx], v0)
            n_mig += 1
    assert n_mig > 0
    for rt in rts:
        _attention_check(rt, shape, q)


class _ThreadHub:
    """torch.distributed's batched P2P for ranks that are threads of one process on one device:
    a sender records an event on its current (copy) stream, the receiver's copy stream waits for
    it and copies — device-asynchronous, like NCCL, so copies can overlap kernels."""

    class P2POp:
        def __init__(self, op, tensor, peer):
            self.op, self.tensor, self.peer = op, tensor, peer

    def __init__(self, world):
        import threading
        self.box, self.bar, self.tls = {}, threading.Barrier(world), threading.local()

    @staticmethod
    def get_backend():
        return "nccl"

    def isend(self):
        pass

    def irecv(self):
        pass

    def batch_isend_irecv(self, ops):
        me = self.tls.rank
        for o in ops:
            if o.op == self.isend:
                ev = torch.cuda.Event()
                ev.record()
                self.box.setdefault((me, o.peer), []).append((o.tensor, ev))
        self.bar.wait()
        for o in ops:
            if o.op == self.irecv:
                t, ev = self.box[(o.peer, me)].pop(0)
                torch.cuda.current_stream().wait_event(ev)
                o.tensor.copy_(t)
        self.bar.wait()

        class _W:
            def wait(self):
                pass
        return [_W() for _ in ops]


def test_bidirectional_precopy_overlaps_next_decode():
    """NEXT#1 on the device: in one step rank 0 pre-copies a request to rank 1 and
    rank 1 pre-copies one to rank 0 (both directions at once), on each rank's copy stream, while
    both ranks run their next decode; the copy segments overlap those decodes (CUDA event
    timeline) and every page arrives with its bytes."""
    import threading
    shape = synth.AttnShape("t", 8, 2)
    sim = pipeline.ClusterSim([(0, 1 << 21, 2)], concurrency=24, seed=3, token_budget=10 ** 9, batch_cap=64)
    hub = _ThreadHub(2)
    ops = [pipeline.DeviceOps(shape, "cuda", seed=r) for r in range(2)]
    rts = [pipeline.RankRuntime(sim, r, 200000, shape, ops[r]) for r in range(2)]
    # the largest resident request of each rank moves to the other one (pre-copy round)
    pick = {}
    for r in range(2):
        rids, Ls = sim.batch(r)
        pick[r] = (int(rids[int(np.argmax(Ls))]), int(Ls.max()))
    ev = pipeline.StepEvents()
    ev.precopies = [(pick[0][0], 0, 1, -(-pick[0][1] // 16)), (pick[1][0], 1, 0, -(-pick[1][1] // 16))]
    snaps = {r: (rts[r].pool["k"][torch.tensor(rts[r].pages[pick[r][0]], device="cuda")].clone(),
                 rts[r].pool["v"][torch.tensor(rts[r].pages[pick[r][0]], device="cuda")].clone()) for r in range(2)}
    q = torch.randn(64, shape.num_q_heads, 128, device="cuda").to(torch.bfloat16)
    # warm-ups: the first launch of a kernel loads its module (lazy loading synchronises the
    # device), and a cudaMalloc inside apply() would too; either would serialise the copy
    for r in range(2):
        kv_len, indptr = rts[r].device_batch()
        l4.decode_attention(q[:len(kv_len)], rts[r].pool["k"], rts[r].pool["v"], torch.from_numpy(indptr).cuda(),
                            rts[r].table, torch.from_numpy(kv_len).cuda())
        l4.pack_pages(rts[r].pool["view"], [0], torch.empty(2 * rts[r].pool["view"].page_bytes, dtype=torch.uint8,
                                                             device="cuda"))
    for r in range(2):
        with torch.cuda.stream(ops[r].copy_stream):
            tmp = [torch.empty(4 * 2 * max(pick[0][1], pick[1][1]) // 16 * rts[r].pool["view"].page_bytes,
                               dtype=torch.uint8, device="cuda") for _ in range(4)]
            del tmp
    torch.cuda.synchronize()
    errs = []

    def rank_main(r):
        try:
            hub.tls.rank = r
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                rt, op = rts[r], ops[r]
                kv_len, indptr = rt.device_batch()       # pre-copies leave the batch unchanged
                B = len(kv_len)
                d_len, d_ptr = (torch.from_numpy(x).cuda() for x in (kv_len, indptr))
                torch.cuda.synchronize()
                for step in range(2):
                    op.before_decode()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    # keep the device ahead of the host (as in a GPU-bound serving loop): the copy
                    # enqueued by apply() starts when this step's decode ends, while the host has
                    # long enqueued the next step's decode
                    # (~100 ms of spinning: the host's apply() of step 0 -- thread-hub barriers, pack
                    # launches -- must finish before this step's decodes end, even on a loaded host)
                    torch.cuda._sleep(200_000_000)
                    for _ in range(4):
                        l4.decode_attention(q[:B], rt.pool["k"], rt.pool["v"], d_ptr, rt.table, d_len)
                    e1.record()
                    op.after_decode(e1, e0)
                    if step == 0:
                        rt.apply(ev, hub)
                op.drain()
                torch.cuda.synchronize()
        except BaseException as e:   # noqa
            errs.append(e)
            hub.bar.abort()

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errs, errs
    for r in range(2):
        st = ops[r].transfer_stats()
        c0, c1, _, _, win = ops[r].timeline[-1]
        rel = None if win is None else [round(c0.elapsed_time(x), 3) for x in (c1, win[0], win[1])]
        assert st["copy_bytes"] > 0 and st["overlap_steps"] == 1, (st, len(ops[r].timeline), rel)
        other = 1 - r
        rid = pick[other][0]
        pages = rts[r].incoming[rid]
        k0, v0 = snaps[other]
        idx = torch.tensor(pages, device="cuda")
        assert torch.equal(rts[r].pool["k"][idx], k0) and torch.equal(rts[r].pool["v"][idx], v0)
