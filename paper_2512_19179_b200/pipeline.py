"""L4 length-aware pipeline over GPUs — host control plane.

  P:255  instances are grouped into length-specialised stages forming a logical pipeline
  P:267  "when a request arrives, it is routed to the earliest stage whose serving range
         covers its initial length ... As the sequence grows, if its length exceeds the
         instance's range, it is migrated to the next stage"
  P:281  the Coordinator "allocates memory on the target instance, and transfers the KV cache"
  P:428  KV goes "directly into idle slots"; migration is skipped if no idle cache is
         available; at most three transfers in flight (excess requests keep running on
         the source)

Each GPU (rank) is one instance.  ``l4_partition`` (the §4.2 DP, host C++) turns a
request-length sample into stages; stage k gets the next ``instances_k`` ranks.

The control plane here is REPLICATED and deterministic: every rank simulates the whole
cluster's request state (ClusterSim) from the same seed, so every rank knows every
routing / handover / retirement decision without exchanging control messages.  The only
cross-GPU traffic is KV-page migration (north star).  The data path of each step — the
decode attention over the local batch and the page pack/unpack — runs in libl4 kernels;
the transport is torch.distributed send/recv (NCCL over NVLink on GPUs).

Within a stage the receiving rank is chosen by the configured policy (least-loaded, the
bid-ask rule of P:395-399, or round-robin).  Boundaries between stages are refined every
``refine_every`` steps (§4.3): each instance calls l4_refine_boundary (host C++) on
the replicated state, so every rank computes the same new boundaries without messages.

Device side (DeviceOps): KV-page transfers run on a dedicated copy stream that waits for the
step's decode and overlaps the next one; a step's decode waits for the copy stream only
when a handed-over request joins this rank's batch.  Pages freed in a step return to the
allocator only after the kernels that may still read them (that step's decode, or the copy
that sends them) have completed.
"""
from __future__ import annotations

import heapq
import math
import time
from dataclasses import dataclass, field
from typing import Dict, List, Tuple

import numpy as np

PAGE = 16


@dataclass
class Req:
    rid: int
    I: int
    O: int
    L: int          # current length (tokens whose KV is cached)
    rank: int


@dataclass
class StepEvents:
    """What happened in one decode step, identical on every rank."""
    # handovers: (rid, src, dst, L at handover, first page to send); first page > 0 is the stop
    # round of a live migration whose earlier pages were pre-copied
    migrations: List[Tuple[int, int, int, int, int]] = field(default_factory=list)
    precopies: List[Tuple[int, int, int, int]] = field(default_factory=list)    # (rid, src, dst, pages)
    cancelled: List[Tuple[int, int]] = field(default_factory=list)             # (rid, dst) live sessions dropped
    retired: List[Tuple[int, int]] = field(default_factory=list)               # (rid, rank)
    admitted: List[Tuple[int, int, int]] = field(default_factory=list)         # (rid, rank, L)
    deferred: int = 0                                                           # handovers over the cap


def detect_overload(my_load: float, stage_loads, factor: float = 1.25) -> bool:
    """an instance is an overloaded outlier when its request-memory demand is more
    than 25% above the stage average (strict, S:399 decision)."""
    loads = list(stage_loads)
    return len(loads) > 0 and my_load > factor * (sum(loads) / len(loads))


def select_receiver(bids):
    """P:395-399 bid-ask: bids = [(receiver, load, earliest_start, reply_time)].  Keep the
    lower-load half (ceil(k/2)), then the three earliest transmission starts, then the one that
    replied first; ties by receiver id at every step."""
    if not bids:
        return None
    half = sorted(bids, key=lambda b: (b[1], b[0]))[: (len(bids) + 1) // 2]
    early = sorted(half, key=lambda b: (b[2], b[0]))[:3]
    return min(early, key=lambda b: (b[3], b[0]))[0]


def assign_ranks(stages) -> List[int]:
    """rank -> stage index: stage k takes the next instances_k ranks (NVSwitch: placement is free)."""
    out = []
    for k, (_, _, m) in enumerate(stages):
        out.extend([k] * m)
    return out


class RequestStream:
    """Deterministic (I, O) source shaped like the paper's ShareGPT traces (synth M5)."""

    def __init__(self, seed: int, max_len: int = 131072, chunk: int = 4096):
        import synth
        self._synth = synth
        self.seed, self.max_len, self.chunk = seed, max_len, chunk
        self._buf: list = []
        self._k = 0
        self.next_rid = 0

    def next(self):
        if not self._buf:
            I, O = self._synth.requests_sharegpt_like(seed=self.seed * 1000003 + self._k, n=self.chunk,
                                                      max_len=self.max_len)
            self._k += 1
            self._buf = list(zip(I.tolist(), O.tolist()))[::-1]
        I, O = self._buf.pop()
        rid = self.next_rid
        self.next_rid += 1
        return rid, int(I), int(O)


class ClusterSim:
    """Replicated, deterministic simulation of the cluster's requests (no GPU state).

    Requests live in slots (numpy arrays); every operation is a deterministic function of
    the seed, so all ranks compute identical states and events.  Per-step work is
    vectorised; only the few handovers / arrivals run Python loops."""

    def __init__(self, stages, concurrency: int, seed: int = 0, token_budget: int = 1_200_000,
                 batch_cap: int = 1024, max_transfers: int = 3, precopy_lead: int = 0,
                 policy: str = "least_loaded", rebalance_every: int = 0, overload_factor: float = 1.25,
                 migrate_Bps: float = 7.7e11, kv_bytes_per_token: int = 131072, refine_every: int = 0,
                 qoe_d=None, refine_alpha: float = 0.3, min_traffic: int = 5):
        self.stages = [(int(lo), int(hi), int(m)) for lo, hi, m in stages]
        # receiver choice within a stage: "least_loaded", "bidask" or "round_robin";
        # intra-stage rebalancing of overloaded instances every `rebalance_every` steps
        assert policy in ("least_loaded", "bidask", "round_robin")
        self.policy = policy
        self.rebalance_every = int(rebalance_every)
        self.overload_factor = float(overload_factor)
        self.migrate_Bps, self.kvb = float(migrate_Bps), int(kv_bytes_per_token)
        self.step_no = 0
        self.queued_tokens = None         # per-rank tokens being handed to it this step (earliest start)
        self._rr = {}
        # NEXT#1 live migration: a request within `precopy_lead` tokens of its stage's upper
        # bound starts a session: its pages are pre-copied to the chosen receiver while it keeps
        # decoding on the source; at the handover only the pages changed since are sent
        # (stop round).  0 = single-round migration at the handover.
        self.precopy_lead = int(precopy_lead)
        self.sessions: Dict[int, list] = {}   # rid -> [src, dst, pages pre-copied]
        self.rank_stage = np.array(assign_ranks(self.stages), dtype=np.int64)
        self.n_ranks = len(self.rank_stage)
        self.stage_hi = np.array([hi for _, hi, _ in self.stages], dtype=np.int64)
        # NEXT#2 adaptive range refinement: every instance owns the upper boundary of
        # its range (initialised from the offline plan), refined every `refine_every`
        # steps from its own and its successors' (I, L) sets; a request hands over when its
        # length reaches its instance's boundary.  Arrivals route by stage bounds = the mean of
        # the stage's instance boundaries (reading Z43).
        self.refine_every = int(refine_every)
        self.qoe_d = tuple(qoe_d) if qoe_d is not None else None
        self.refine_alpha, self.min_traffic = float(refine_alpha), int(min_traffic)
        self.rank_hi = self.stage_hi[self.rank_stage].astype(np.float64)
        self.bounds = self.stage_hi.astype(np.float64)           # routing upper bound per stage
        self._bounds_l = self.bounds.tolist()[: len(self.stages) - 1]   # (Python copy for stage_of)
        self.refinements = 0
        self.last_stage = len(self.stages) - 1
        self.stage_ranks = [[r for r in range(self.n_ranks) if self.rank_stage[r] == k] for k in range(len(self.stages))]
        self.token_budget = token_budget      # admission limit per instance (KV memory)
        self.batch_cap = batch_cap
        self.max_transfers = max_transfers
        self.stream = RequestStream(seed)
        self.rng = np.random.default_rng(seed + 17)
        cap = max(16, 2 * concurrency + self.n_ranks * 4)
        self.rid = np.full(cap, -1, dtype=np.int64)
        self.I = np.zeros(cap, dtype=np.int64)
        self.O = np.zeros(cap, dtype=np.int64)
        self.L = np.zeros(cap, dtype=np.int64)
        self.rank = np.full(cap, -1, dtype=np.int64)
        self.active = np.zeros(cap, dtype=bool)
        self._free = list(range(cap))         # free slots, a min-heap: placement takes the lowest
        self.tokens = np.zeros(self.n_ranks, dtype=np.int64)
        self.count = np.zeros(self.n_ranks, dtype=np.int64)
        self.queue: List[Tuple[int, int, int]] = []
        for _ in range(concurrency):          # stationary start: a random point of each lifetime
            rid, I, O = self.stream.next()
            L = I + int(self.rng.integers(0, O))
            self._place(rid, I, O, L, initial=True)

    @property
    def reqs(self):
        """rid -> Req view (diagnostics / tests)."""
        idx = np.nonzero(self.active)[0]
        return {int(self.rid[i]): Req(int(self.rid[i]), int(self.I[i]), int(self.O[i]), int(self.L[i]),
                                      int(self.rank[i])) for i in idx}

    # ---------------------------------------------------------------- routing
    def stage_of(self, L: int) -> int:
        """Earliest stage whose range covers length L; the last stage takes the rest."""
        for k, b in enumerate(self._bounds_l):
            if L < b:
                return k
        return self.last_stage

    def current_stages(self):
        """(lo, hi, instances) with the current (refined) routing bounds, rounded down."""
        out, lo = [], 0
        for k, (_, hi, m) in enumerate(self.stages):
            h = int(hi) if k == self.last_stage else int(math.floor(self.bounds[k]))
            out.append((lo, h, m))
            lo = h
        return out

    def _fits(self, r: int, extra_tokens: int) -> bool:
        return self.count[r] < self.batch_cap and self.tokens[r] + extra_tokens <= self.token_budget

    def least_loaded(self, stage: int, extra_tokens: int = 0, exclude: int = -1):
        """Receiver of a request in `stage` under the configured policy; instances without
        idle KV capacity abstain."""
        cands = [r for r in self.stage_ranks[stage] if r != exclude and self._fits(r, extra_tokens)]
        if not cands:
            return None
        if self.policy == "round_robin":
            k = self._rr.get(stage, 0)
            order = self.stage_ranks[stage]
            for t in range(len(order)):
                r = order[(k + t) % len(order)]
                if r in cands:
                    self._rr[stage] = (k + t + 1) % len(order)
                    return r
        if self.policy == "bidask":
            q = self.queued_tokens
            bids = []
            for r in cands:
                start = (0.0 if q is None else float(q[r])) * self.kvb / self.migrate_Bps   # earliest start (s)
                reply = ((self.step_no * 1000003 + r * 7919 + extra_tokens * 31) % 1009) / 1009.0  # deterministic
                bids.append((r, int(self.tokens[r]), start, reply))
            return select_receiver(bids)
        best = None
        for r in cands:
            if best is None or self.tokens[r] < self.tokens[best]:
                best = r
        return best

    def _free_slot(self):
        """The lowest free slot (a min-heap of free slots; the arrays double when none is left)."""
        if not self._free:
            n = self.rid.size
            for name in ("rid", "I", "O", "L", "rank"):
                arr = getattr(self, name)
                fill = -1 if name in ("rid", "rank") else 0
                setattr(self, name, np.concatenate([arr, np.full(n, fill, dtype=arr.dtype)]))
            self.active = np.concatenate([self.active, np.zeros(n, dtype=bool)])
            self._free = list(range(n, 2 * n))
        return heapq.heappop(self._free)

    def _place(self, rid, I, O, L, initial=False, fail_cache=None):
        k = self.stage_of(L)
        # within one arrivals pass capacity only shrinks, so once no instance of stage k fits
        # `extra` tokens, none fits more (exact shortcut for the queued retries)
        if fail_cache is not None and L + 1 >= fail_cache.get(k, 1 << 62):
            r = None
        else:
            r = self.least_loaded(k, L + 1)
            if r is None and fail_cache is not None:
                fail_cache[k] = min(fail_cache.get(k, 1 << 62), L + 1)
        if r is None:
            if not initial:
                self.queue.append((rid, I, O))
            return None
        i = self._free_slot()
        self.rid[i], self.I[i], self.O[i], self.L[i], self.rank[i], self.active[i] = rid, I, O, L, r, True
        self.tokens[r] += L
        self.count[r] += 1
        return r

    # ---------------------------------------------------------------- one decode step
    def step(self) -> StepEvents:
        ev = StepEvents()
        self.step_no += 1
        self.queued_tokens = np.zeros(self.n_ranks, dtype=np.int64)
        act = self.active
        # 1. every resident request generated one token: its KV grows by one
        self.L[act] += 1
        self.tokens += np.bincount(self.rank[act], minlength=self.n_ranks)
        # 2. retire finished requests (closed loop: each is replaced by an arrival)
        done = np.nonzero(act & (self.L >= self.I + self.O))[0]
        for i in done:
            r = int(self.rank[i])
            ev.retired.append((int(self.rid[i]), r))
            self.tokens[r] -= self.L[i]
            self.count[r] -= 1
            self.active[i] = False
            heapq.heappush(self._free, int(i))
        # 2b. live sessions of retired requests are dropped (the receiver frees its copy)
        for rid, r in ev.retired:
            ses = self.sessions.pop(rid, None)
            if ses is not None:
                ev.cancelled.append((rid, ses[1]))
        # 3. handover to the next stage when the length leaves the stage range
        act = self.active
        st = self.rank_stage[np.maximum(self.rank, 0)]
        nonlast = act & (st != self.last_stage)
        hi = self.rank_hi[np.maximum(self.rank, 0)]               # the instance's own boundary
        cand = np.nonzero(nonlast & (self.L >= hi))[0]
        inflight = np.zeros(self.n_ranks, dtype=np.int64)   # transfers in flight per sender
        for ses in self.sessions.values():
            inflight[ses[0]] += 1
        for i in cand:                       # slot order: deterministic on every rank
            rid, src, L = int(self.rid[i]), int(self.rank[i]), int(self.L[i])
            ses = self.sessions.pop(rid, None)
            if ses is not None:                        # stop round of a live migration
                dst, first = ses[1], max(ses[2] - 1, 0)
                inflight[src] -= 1
            else:
                if inflight[src] >= self.max_transfers:    # keep running on the source
                    ev.deferred += 1
                    continue
                dst = self.least_loaded(self.next_stage(int(self.rank_stage[src]), L), L)
                if dst is None:                            # no idle cache downstream: skip
                    ev.deferred += 1
                    continue
                first = 0
                inflight[src] += 1                          # single-round transfer this step
            self._move(i, src, dst, L)
            ev.migrations.append((rid, src, dst, L, first))
        # 3b. live migration: start pre-copy rounds for requests about to leave their range
        if self.precopy_lead > 0:
            near = np.nonzero(nonlast & self.active & (self.L < hi) & (self.L >= hi - self.precopy_lead))[0]
            for i in near:
                rid, src, L = int(self.rid[i]), int(self.rank[i]), int(self.L[i])
                if rid in self.sessions or inflight[src] >= self.max_transfers:
                    continue
                dst = self.least_loaded(self.next_stage(int(self.rank_stage[src]), int(math.ceil(hi[i]))),
                                        L + self.precopy_lead)
                if dst is None:
                    continue
                npg = -(-L // PAGE)
                self.sessions[rid] = [src, dst, npg]
                inflight[src] += 1
                ev.precopies.append((rid, src, dst, npg))
        # 3c. intra-stage rebalancing of overloaded instances via bid-ask
        if self.rebalance_every > 0 and self.step_no % self.rebalance_every == 0:
            self._rebalance(ev, inflight)
        # 3d. adaptive range refinement
        if self.refine_every > 0 and self.step_no % self.refine_every == 0:
            self.refine()
        # 4. arrivals: queued first, then one new request per retirement
        pending, self.queue = self.queue, []
        for _ in range(len(done)):
            pending.append(self.stream.next())
        fail_cache = {}
        for rid, I, O in pending:
            r = self._place(rid, I, O, I, fail_cache=fail_cache)
            if r is not None:
                ev.admitted.append((rid, r, I))
        return ev

    def next_stage(self, k: int, L: int) -> int:
        """Destination stage of a request leaving stage k with length L: the next stage, or a
        later one when L already lies beyond it."""
        return min(self.last_stage, max(k + 1, self.stage_of(L)))

    def refine(self):
        """§4.3 on every instance of every non-last stage: l4_refine_boundary over the
        instance's (I, L) list and its successors' (the next stage's instances), EMA-smoothed and
        frozen below `min_traffic` requests; the result clamps to (stage lo, successor hi).  The
        same host code on the same replicated state gives every rank the same boundaries."""
        from . import l4
        if self.qoe_d is None:
            import synth
            self.qoe_d = synth.roofline_qoe_d()
        act = np.nonzero(self.active)[0]
        per_rank = [[] for _ in range(self.n_ranks)]
        for i in act:
            per_rank[int(self.rank[i])].append((int(self.I[i]), int(self.L[i])))
        new_hi = self.rank_hi.copy()
        for k in range(self.last_stage):
            lo = 0 if k == 0 else int(math.floor(self.bounds[k - 1]))
            hi = int(self.stage_hi[-1]) if k + 1 == self.last_stage else int(math.ceil(self.bounds[k + 1]))
            if hi - lo < 2:
                continue
            succ = [per_rank[r] for r in self.stage_ranks[k + 1]]
            for r in self.stage_ranks[k]:
                nb, _, _ = l4.refine_boundary(float(self.rank_hi[r]), per_rank[r], succ, self.qoe_d,
                                              alpha=self.refine_alpha, min_traffic=self.min_traffic, lo=lo, hi=hi)
                new_hi[r] = nb
        self.rank_hi = new_hi
        for k in range(self.last_stage):
            self.bounds[k] = float(np.mean([self.rank_hi[r] for r in self.stage_ranks[k]]))
        self._bounds_l = self.bounds.tolist()[: self.last_stage]
        self.refinements += 1

    def _move(self, i, src, dst, L):
        self.tokens[src] -= L
        self.count[src] -= 1
        self.rank[i] = dst
        self.tokens[dst] += L
        self.count[dst] += 1
        self.queued_tokens[dst] += L

    def _rebalance(self, ev, inflight):
        """An instance whose load exceeds 1.25x its stage mean hands requests (largest first,
        slot order on ties) to bid-ask winners among its stage peers until it is no longer an
        outlier or its transfer cap is reached."""
        for k, ranks in enumerate(self.stage_ranks):
            if len(ranks) < 2:
                continue
            for src in ranks:
                loads = [int(self.tokens[r]) for r in ranks]
                if not detect_overload(int(self.tokens[src]), loads, self.overload_factor):
                    continue
                mine = np.nonzero(self.active & (self.rank == src))[0]
                mine = sorted(mine.tolist(), key=lambda i: (-int(self.L[i]), i))
                mean = sum(loads) / len(loads)
                for i in mine:
                    if inflight[src] >= self.max_transfers or self.tokens[src] <= mean:
                        break
                    rid, L = int(self.rid[i]), int(self.L[i])
                    if rid in self.sessions:
                        continue
                    dst = self.least_loaded(k, L, exclude=src)
                    if dst is None or self.tokens[dst] + L >= self.tokens[src]:
                        continue                    # would not reduce the imbalance
                    self._move(i, src, dst, L)
                    inflight[src] += 1
                    ev.migrations.append((rid, src, dst, L, 0))

    def stage_cv(self):
        """Per-stage coefficient of variation of resident tokens (Fig. 16 metric)."""
        out = []
        for ranks in self.stage_ranks:
            if len(ranks) < 2:
                continue
            x = np.array([self.tokens[r] for r in ranks], dtype=np.float64)
            out.append(float(x.std() / x.mean()) if x.mean() > 0 else 0.0)
        return out

    def batch(self, rank: int):
        """Resident requests of a rank in slot order: (rid array, L array)."""
        idx = np.nonzero(self.active & (self.rank == rank))[0]
        return self.rid[idx], self.L[idx]

    def fingerprint(self) -> int:
        idx = np.nonzero(self.active)[0]
        order = np.argsort(self.rid[idx])
        data = np.stack([self.rid[idx][order], self.L[idx][order], self.rank[idx][order]]).astype(np.int64)
        h = 1469598103934665603
        for x in data.ravel().tolist() + self.rank_hi.view(np.int64).tolist():
            h = ((h ^ (x & 0xFFFFFFFF)) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
        return h


def plan_stages(n_instances: int, seed: int = 0, n_sample: int = 10000, qoe_d=None,
                bandwidth_Bps: float = 7.7e11, kv_bytes_per_token: int = 131072, mode: int = 0):
    """l4_partition over a request sample (the period's statistics)."""
    import synth
    from . import l4
    I, O = synth.requests_sharegpt_like(seed=seed, n=n_sample)
    D = synth.roofline_qoe_d() if qoe_d is None else qoe_d
    stages, obj = l4.partition(I, O, n_instances, D, bandwidth_Bps, kv_bytes_per_token, mode=mode)
    return stages, obj


class RankRuntime:
    """One rank's device state: a paged KV pool (one layer materialised), the page tables of
    its resident requests, and the per-step data path (attention + migration transport).

    Page tables live on the device as a block table [slots, max_pages] (row = one resident
    request, fixed stride), so the decode kernel gets indptr[b] = slot_b * max_pages and no
    CSR is rebuilt per step; the host sends only the per-step page-id deltas.
    ``ops`` provides the device operations (DeviceOps: libl4 on CUDA).
    """

    def __init__(self, sim: ClusterSim, rank: int, num_pages: int, shape, ops, seed: int = 0,
                 max_pages_per_req: int = 131072 // PAGE):
        self.sim, self.rank, self.shape, self.ops = sim, rank, shape, ops
        self.num_pages = num_pages
        self.pool = ops.make_pool(num_pages)
        self.max_pages = max_pages_per_req
        self.slots_cap = sim.batch_cap
        self.table = ops.make_table(self.slots_cap, self.max_pages) if hasattr(ops, "make_table") else None
        self.free_slots = list(range(self.slots_cap))[::-1]
        self.slot_of: Dict[int, int] = {}
        self.pages: Dict[int, List[int]] = {}
        self._dpos: List[np.ndarray] = []
        self._dval: List[np.ndarray] = []
        rids, Ls = sim.batch(rank)
        for rid, L in zip(rids.tolist(), Ls.tolist()):
            self._add(rid, ops.alloc(self.pool, -(-L // PAGE)))
        self.incoming: Dict[int, List[int]] = {}   # live migration: pages pre-copied to this rank
        self.stats = dict(migrated_pages=0, migrated_bytes=0, migrations_in=0, migrations_out=0, launches=0,
                          precopy_pages=0, stop_pages=0, single_pages=0)

    # ------------------------------------------------------------ page-table bookkeeping
    def _delta(self, slot, start, pages):
        if pages:
            self._dpos.append(slot * self.max_pages + start + np.arange(len(pages), dtype=np.int64))
            self._dval.append(np.asarray(pages, dtype=np.int32))

    def _add(self, rid, pages):
        slot = self.free_slots.pop()
        self.slot_of[rid] = slot
        self.pages[rid] = list(pages)
        self._delta(slot, 0, self.pages[rid])

    def _append(self, rid, new_pages):
        start = len(self.pages[rid])
        self.pages[rid].extend(new_pages)
        self._delta(self.slot_of[rid], start, new_pages)

    def _drop(self, rid):
        self.free_slots.append(self.slot_of.pop(rid))
        return self.pages.pop(rid)

    def device_batch(self):
        """(kv_len int32 [B], indptr int32 [B+1]) of the resident batch in slot-table form,
        after flushing this step's page-table deltas to the device table."""
        if self._dpos:
            self.ops.table_update(self.table, np.concatenate(self._dpos), np.concatenate(self._dval))
            self._dpos, self._dval = [], []
        rids, Ls = self.sim.batch(self.rank)
        slots = np.fromiter((self.slot_of[r] for r in rids.tolist()), dtype=np.int64, count=len(rids))
        indptr = np.empty(len(rids) + 1, dtype=np.int32)
        indptr[:-1] = slots * self.max_pages
        indptr[-1] = self.slots_cap * self.max_pages
        return Ls.astype(np.int32), indptr

    def tables(self):
        """Compact host CSR of the resident batch (tests / diagnostics)."""
        rids, Ls = self.sim.batch(self.rank)
        kv_len = Ls.astype(np.int32)
        lists = [self.pages[rid] for rid in rids.tolist()]
        counts = np.fromiter((len(x) for x in lists), dtype=np.int64, count=len(lists))
        indptr = np.zeros(len(lists) + 1, dtype=np.int32)
        indptr[1:] = np.cumsum(counts)
        indices = (np.fromiter((p for x in lists for p in x), dtype=np.int32, count=int(indptr[-1]))
                   if lists else np.zeros(0, dtype=np.int32))
        return kv_len, indptr, indices

    def reset_stats(self):
        for k in self.stats:
            self.stats[k] = 0
        if hasattr(self.ops, "reset_transfer_stats"):
            self.ops.reset_transfer_stats()

    def apply(self, ev: StepEvents, comm):
        """Apply one step's events to this rank: retire, grow page lists (new tokens),
        migrate KV pages out/in (P2P), admit new requests."""
        nvtx = getattr(getattr(getattr(self.ops, "torch", None), "cuda", None), "nvtx", None)
        if nvtx is not None:
            nvtx.range_push("l4.pipeline.apply")
        try:
            self._apply(ev, comm)
        finally:
            if nvtx is not None:
                nvtx.range_pop()

    def _apply(self, ev: StepEvents, comm):
        me = self.rank
        free_sent = getattr(self.ops, "free_after_transfer", self.ops.free)
        for rid, r in ev.retired:
            if r == me and rid in self.pages:
                self.ops.free(self.pool, self._drop(rid))
        # growth: the step's new token opens a new page when L-1 is a multiple of 16
        sim = self.sim
        mig_out = {m[0] for m in ev.migrations if m[1] == me} | {p[0] for p in ev.precopies if p[1] == me}
        mine = sim.rank == me
        if mig_out:
            mine = mine | np.isin(sim.rid, np.fromiter(mig_out, dtype=np.int64, count=len(mig_out)))
        grow = np.nonzero(sim.active & mine & ((sim.L - 1) % PAGE == 0))[0]
        wants = []
        for rid, L in zip(sim.rid[grow].tolist(), sim.L[grow].tolist()):
            if rid in self.pages:
                n = -(-L // PAGE) - len(self.pages[rid])
                if n > 0:
                    wants.append((rid, n))
        if wants:  # one lowest-free-first allocation for all of them, dealt out in the same order
            got = self.ops.alloc(self.pool, sum(n for _, n in wants))
            o = 0
            for rid, n in wants:
                self._append(rid, got[o:o + n])
                o += n
        for rid, dst in ev.cancelled:                 # live session of a retired request
            if dst == me and rid in self.incoming:
                self.ops.free(self.pool, self.incoming.pop(rid))
        # transfers in global event order: pre-copy rounds, then handovers (single or stop round)
        sends, recvs, done_out, done_in = [], [], [], []
        for rid, src, dst, npg in ev.precopies:
            if src == me:
                sends.append((dst, self.pages[rid][:npg]))
                self.stats["precopy_pages"] += npg
            elif dst == me:
                pages = self.ops.alloc(self.pool, npg)
                self.incoming[rid] = pages
                recvs.append((src, pages))
        for rid, src, dst, L, first in ev.migrations:
            need = -(-L // PAGE)
            if src == me:
                pages = self._drop(rid)
                if need > len(pages):
                    pages = pages + self.ops.alloc(self.pool, need - len(pages))
                sends.append((dst, pages[first:need]))
                done_out.append(pages)
                self.stats["stop_pages" if first > 0 else "single_pages"] += need - first
            elif dst == me:
                have = self.incoming.pop(rid, [])[:first + 1] if first > 0 else []
                if first > 0:
                    pages = have[:first] + (have[first:first + 1] or self.ops.alloc(self.pool, 1))
                else:
                    pages = []
                pages = pages + self.ops.alloc(self.pool, need - len(pages))
                recvs.append((src, pages[first:need]))
                done_in.append((rid, pages))
        nbytes = self.ops.transfer(self.pool, sends, recvs, comm, any_transfer=bool(ev.precopies or ev.migrations),
                                   joins=len(done_in), sent=len(done_out))
        for rid, pages in done_in:
            self._add(rid, pages)
        for pages in done_out:
            free_sent(self.pool, pages)
            self.stats["migrations_out"] += 1
            self.stats["migrated_pages"] += len(pages)
        self.stats["migrations_in"] += len(done_in)
        self.stats["migrated_bytes"] += nbytes
        self.stats["launches"] += len(sends) + len(recvs)
        for rid, r, L in ev.admitted:
            if r == me:
                self._add(rid, self.ops.alloc(self.pool, -(-L // PAGE)))   # prefill not emulated


class H2DRing:
    """Small per-step host->device copies without per-step pinned allocations: a ring of
    preallocated pinned host buffers and device buffers; several int32 arrays are packed into
    one slot and moved with one async copy on the current stream.  A slot is reused only after
    its previous copy completed (event).  Arrays larger than a slot take the plain path."""

    def __init__(self, device, slot_bytes: int = 1 << 20, depth: int = 16):
        import torch
        self.torch, self.device, self.slot_bytes, self.depth = torch, device, slot_bytes, depth
        self.h = [torch.empty(slot_bytes, dtype=torch.uint8).pin_memory() for _ in range(depth)]
        self.d = [torch.empty(slot_bytes, dtype=torch.uint8, device=device) for _ in range(depth)]
        self.ev = [None] * depth
        self.i = 0
        self.wait_s = 0.0   # host time spent waiting for a slot's previous copy (device behind)

    def put(self, *arrays):
        torch = self.torch
        arrays = [np.ascontiguousarray(a, dtype=np.int32) for a in arrays]
        offs, off = [], 0
        for a in arrays:
            offs.append(off)
            off += (a.nbytes + 255) // 256 * 256
        if off > self.slot_bytes:
            return [torch.from_numpy(a).to(self.device) for a in arrays]
        k = self.i % self.depth
        self.i += 1
        if self.ev[k] is not None:
            t0 = time.perf_counter()
            self.ev[k].synchronize()
            self.wait_s += time.perf_counter() - t0
        hv = self.h[k].numpy()
        for a, o in zip(arrays, offs):
            hv[o:o + a.nbytes] = a.view(np.uint8)
        self.d[k][:off].copy_(self.h[k][:off], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        self.ev[k] = ev
        return [self.d[k][o:o + a.nbytes].view(torch.int32) for a, o in zip(arrays, offs)]


class DeviceOps:
    """libl4 on CUDA: page pool (host allocator over a device KV pool), attention, and the
    KV-page transport (l4_pack_pages -> NCCL send/recv -> l4_unpack_pages, or one-sided
    l4_copy_pages pushes over CUDA IPC) on a dedicated copy stream.

    Ordering (NEXT#1): the copy stream first waits for everything enqueued on the compute
    stream so far (this step's decode and token writes), so a transfer overlaps the NEXT step's
    decode; that decode waits for the copy stream only when a handed-over request joins this
    rank's batch (before_decode).  Freed pages are returned to the allocator only after the
    event that covers their last reader completed: this step's decode (after_decode) for retired
    requests, the copy for pages that were sent (a receiver writes into idle slots only)."""

    def __init__(self, shape, device, seed=0):
        import torch
        from . import l4
        self.torch, self.l4, self.shape, self.device = torch, l4, shape, device
        self.seed = seed
        self.h2d = H2DRing(device)
        self.copy_stream = torch.cuda.Stream(device=device)
        self.decode_ev = None          # event after the current step's decode (after_decode)
        self.copy_ev = None            # event after the last transfer on the copy stream
        self.join_wait = False         # the next decode must wait for the copy stream
        self.keep = []                 # (event, buffers) staging kept alive until the copy completed
        self.timeline = []             # (copy start, copy end, bytes, joins, decode-end event of the step)
        self.peer_events = {}          # IPC transport: peers' interprocess events
        self.pending_peers = set()

    def make_pool(self, num_pages):
        torch = self.torch
        s = self.shape
        g = torch.Generator(device=self.device).manual_seed(self.seed)
        k = torch.empty(num_pages, s.num_kv_heads, PAGE, s.head_dim, dtype=torch.bfloat16, device=self.device)
        v = torch.empty_like(k)
        for x in (k, v):
            for a in range(0, num_pages, 8192):
                e = min(num_pages, a + 8192)
                x[a:e] = torch.randn(e - a, *x.shape[1:], device=self.device, generator=g).to(torch.bfloat16)
        return dict(k=k, v=v, alloc=self.l4.PagePool(num_pages), view=self.l4.kv_view(k, v), pending=[])

    # ---------------------------------------------------------------- page ownership
    def _reclaim(self, pool, block=False):
        keep = []
        for ev, pages in pool["pending"]:
            if ev is None or ev.query() or block:
                if block and ev is not None:
                    ev.synchronize()
                pool["alloc"].free(pages)
            else:
                keep.append((ev, pages))
        pool["pending"] = keep

    def alloc(self, pool, n):
        self._reclaim(pool)
        try:
            return pool["alloc"].alloc(n).tolist()
        except self.l4.NoPagesError:
            self._reclaim(pool, block=True)        # wait for the readers of the deferred pages
            return pool["alloc"].alloc(n).tolist()

    def free(self, pool, pages):
        """Pages of a retired request: reusable once this step's decode (which read them) completed."""
        if pages:
            pool["pending"].append((self.decode_ev, list(pages)))

    def free_after_transfer(self, pool, pages):
        """Pages sent to another instance: reusable once the copy that reads them completed."""
        if pages:
            pool["pending"].append((self.copy_ev if self.copy_ev is not None else self.decode_ev, list(pages)))

    def make_table(self, slots, max_pages):
        return self.torch.zeros(slots * max_pages, dtype=self.torch.int32, device=self.device)

    def table_update(self, table, pos, val):
        """Scatter this step's page-id deltas into the device block table (pinned H2D, async)."""
        p, v = self.h2d.put(pos, val)
        table.index_copy_(0, p.long(), v)

    # ---------------------------------------------------------------- step hooks (bench loop)
    def before_decode(self):
        """The step's decode waits for pages that landed for requests joining this rank."""
        cur = self.torch.cuda.current_stream(self.device)
        if self.join_wait and self.copy_ev is not None:
            cur.wait_event(self.copy_ev)
        for src in sorted(self.pending_peers):     # IPC: the senders' copy streams
            cur.wait_event(self.peer_events[src])
        self.join_wait = False
        self.pending_peers = set()

    def after_decode(self, ev, ev_start=None):
        """`ev` is recorded after this step's decode (and `ev_start` before it): frees of this
        step wait for it, and the previous step's copy segment is matched to this decode window."""
        self.decode_ev = ev
        if ev_start is not None and self.timeline and self.timeline[-1][4] is None:
            self.timeline[-1][4] = (ev_start, ev)
        self.keep = [(e, b) for e, b in self.keep if not e.query()]

    def drain(self):
        self.copy_stream.synchronize()
        self.torch.cuda.current_stream(self.device).wait_stream(self.copy_stream)

    def reset_transfer_stats(self):
        self.timeline = []

    def transfer_stats(self):
        """Copy-stream timing of the transfers since the last reset: per step with a transfer, the
        copy segment (start..end) against the NEXT step's decode window on the compute stream."""
        out = dict(copy_ms_sum=0.0, copy_bytes=0, stall_ms_sum=0.0, stall_count=0, stall_ms_max=0.0,
                   overlap_steps=0)
        for i, (c0, c1, nb, joins, d_next) in enumerate(self.timeline):
            dt = c0.elapsed_time(c1)
            out["copy_ms_sum"] += dt
            out["copy_bytes"] += nb
            if joins:                           # a handed-over request waits for this segment
                out["stall_ms_sum"] += dt
                out["stall_count"] += joins
                out["stall_ms_max"] = max(out["stall_ms_max"], dt)
            if d_next is not None:
                d0, d1 = d_next
                if c0.elapsed_time(d1) > 0 and d0.elapsed_time(c1) > 0:   # copy window meets next decode
                    out["overlap_steps"] += 1
        return out

    def _segment_begin(self):
        torch = self.torch
        cs = self.copy_stream
        cs.wait_stream(torch.cuda.current_stream(self.device))     # after this step's decode / writes
        c0 = torch.cuda.Event(enable_timing=True)
        c0.record(cs)
        return c0

    def _segment_end(self, c0, nbytes, joins, stalled=None):
        """Close a copy-stream segment; `joins` > 0: the next decode must wait for it; `stalled`:
        handed-over requests whose stop round this segment carries (the stall statistic)."""
        stalled = joins if stalled is None else stalled
        torch = self.torch
        c1 = torch.cuda.Event(enable_timing=True)
        c1.record(self.copy_stream)
        self.copy_ev = c1
        if joins:
            self.join_wait = True
        self.timeline.append([c0, c1, nbytes, int(stalled), None])

    # ---------------------------------------------------------------- one-sided (CUDA IPC)
    def setup_ipc(self, pool, rank: int, world: int, group=None):
        """Map every peer's KV pools into this process (CUDA IPC; handles + offsets travel over
        the CPU process group `group`), and exchange interprocess events that mark the end of each
        peer's pushes.  Afterwards transfer() pushes pages one-sidedly."""
        import torch.distributed as dist
        torch, l4 = self.torch, self.l4
        hk, ok = l4.ipc_get_handle(pool["k"].data_ptr())
        hv, ov = l4.ipc_get_handle(pool["v"].data_ptr())
        self.my_ipc_event = torch.cuda.Event(interprocess=True)
        self.my_ipc_event.record(self.copy_stream)
        mine = (hk, ok, hv, ov, bytes(self.my_ipc_event.ipc_handle()))
        peers = [None] * world
        dist.all_gather_object(peers, mine, group=group)
        view = pool["view"]
        self.ipc_group, self.ipc_rank, self.ipc_views, self.ipc_bases = group, rank, {}, []
        for r, (pk, pok, pv, pov, pev) in enumerate(peers):
            if r == rank:
                continue
            bk, bv = l4.ipc_open_handle(pk), l4.ipc_open_handle(pv)
            self.ipc_bases += [bk, bv]
            self.ipc_views[r] = l4.kv_view(None, None, device=view.device, num_layers=view.num_layers,
                                           num_pages=view.num_pages, layer_stride_bytes=view.layer_stride_bytes,
                                           page_bytes=view.page_bytes, k_ptr=bk + pok, v_ptr=bv + pov)
            self.peer_events[r] = torch.cuda.Event.from_ipc_handle(self.device, pev)

    def close_ipc(self):
        self.drain()
        for b in getattr(self, "ipc_bases", []):
            self.l4.ipc_close_handle(b)
        self.ipc_bases, self.ipc_views = [], {}

    def _transfer_ipc(self, pool, sends, recvs, any_transfer, joins, sent):
        """One-sided: the receivers' destination page lists (allocated in their idle slots)
        reach the senders over the CPU group; each sender writes its pages straight into the
        receiver's pool on its copy stream (l4_copy_pages over the IPC mapping; NVLink across GPUs,
        P:426) and records its interprocess event; a barrier publishes the records, and a receiver
        whose batch gains a handed-over request makes its next decode wait for those senders'
        events.  Every rank takes part whenever any rank transfers."""
        import torch.distributed as dist
        if not any_transfer:
            return 0
        lists = [None] * dist.get_world_size(self.ipc_group)
        dist.all_gather_object(lists, [(src, list(pages)) for src, pages in recvs], group=self.ipc_group)
        me = self.ipc_rank
        queue = {}  # (sender, receiver) -> receiver's destination lists, in event order
        for r, lst in enumerate(lists):
            for src, pages in lst:
                queue.setdefault((src, r), []).append(pages)
        pb = pool["view"].page_bytes
        nbytes = 0
        c0 = self._segment_begin()
        with self.torch.cuda.stream(self.copy_stream):
            for dst, pages in sends:
                dpages = queue[(me, dst)].pop(0)
                assert len(dpages) == len(pages)
                if pages:
                    self.l4.copy_pages(pool["view"], pages, self.ipc_views[dst], dpages, stream=self.copy_stream)
                nbytes += len(pages) * 2 * pb
            self.my_ipc_event.record(self.copy_stream)
        self._segment_end(c0, nbytes, 0, stalled=sent)   # the sender's segment carries the stop rounds
        nbytes += sum(len(p) for _, p in recvs) * 2 * pb
        dist.barrier(group=self.ipc_group)                 # every sender recorded its event
        if joins:
            self.pending_peers |= {src for src, pages in recvs if pages}
        return nbytes

    def transfer(self, pool, sends, recvs, comm, any_transfer=None, joins=0, sent=0):
        """sends = [(dst rank, src page ids)], recvs = [(src rank, dst page ids)] in the global
        event order: pack -> batched NCCL P2P -> unpack straight into the receiver's pages
        (allocated by the caller in idle slots), on the copy stream, or the one-sided IPC
        push after setup_ipc().  joins: handed-over requests entering this rank's batch next step
        (their decode waits for this copy); sent: handed-over requests this rank sends.
        Returns bytes moved by this rank."""
        torch, l4, dist = self.torch, self.l4, comm
        if getattr(self, "ipc_views", None) is not None and hasattr(self, "ipc_rank"):
            return self._transfer_ipc(pool, sends, recvs,
                                      any_transfer if any_transfer is not None else bool(sends or recvs), joins, sent)
        if not sends and not recvs:
            return 0
        pb = pool["view"].page_bytes
        # NCCL moves device buffers over NVLink; the gloo backend (development: several ranks
        # sharing one GPU) needs host buffers, so the staging goes through host memory there.
        host = dist.get_backend() == "gloo"
        ops, bufs, keep, nbytes = [], [], [], 0
        c0 = self._segment_begin()
        cs = self.copy_stream
        with torch.cuda.stream(cs):
            for dst, pages in sends:
                st = torch.empty(max(len(pages), 1) * 2 * pb, dtype=torch.uint8, device=self.device)
                if pages:
                    l4.pack_pages(pool["view"], pages, st, stream=cs)
                ops.append(dist.P2POp(dist.isend, st.cpu() if host else st, dst))
                keep.append(st)
                nbytes += len(pages) * 2 * pb
            for src, pages in recvs:
                st = torch.empty(max(len(pages), 1) * 2 * pb, dtype=torch.uint8, device="cpu" if host else self.device)
                ops.append(dist.P2POp(dist.irecv, st, src))
                bufs.append((pages, st))
                keep.append(st)
                nbytes += len(pages) * 2 * pb
            for w in dist.batch_isend_irecv(ops):
                w.wait()                         # NCCL: the copy stream waits; the host does not
            for pages, st in bufs:
                if pages:
                    l4.unpack_pages(pool["view"], pages, st.to(self.device) if host else st, stream=cs)
        self._segment_end(c0, nbytes, joins)
        self.keep.append((self.copy_ev, keep))   # staging buffers live until the copy completed
        return nbytes
