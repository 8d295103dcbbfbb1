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

Within a stage the receiving rank is the least-loaded one by resident tokens (a simple
stand-in for the bid-ask protocol, which is a next step).
"""
from __future__ import annotations

import math
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
                 migrate_Bps: float = 7.7e11, kv_bytes_per_token: int = 131072):
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
        for k, (lo, hi, _) in enumerate(self.stages):
            if lo <= L < hi:
                return k
        return self.last_stage

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
        free = np.nonzero(~self.active)[0]
        if free.size == 0:
            n = self.rid.size
            for name in ("rid", "I", "O", "L", "rank"):
                arr = getattr(self, name)
                fill = -1 if name in ("rid", "rank") else 0
                setattr(self, name, np.concatenate([arr, np.full(n, fill, dtype=arr.dtype)]))
            self.active = np.concatenate([self.active, np.zeros(n, dtype=bool)])
            return n
        return int(free[0])

    def _place(self, rid, I, O, L, initial=False):
        r = self.least_loaded(self.stage_of(L), L + 1)
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
        # 2b. live sessions of retired requests are dropped (the receiver frees its copy)
        for rid, r in ev.retired:
            ses = self.sessions.pop(rid, None)
            if ses is not None:
                ev.cancelled.append((rid, ses[1]))
        # 3. handover to the next stage when the length leaves the stage range
        act = self.active
        st = self.rank_stage[np.maximum(self.rank, 0)]
        nonlast = act & (st != self.last_stage)
        hi = self.stage_hi[st]
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
                dst = self.least_loaded(self.stage_of(L), L)
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
                dst = self.least_loaded(self.stage_of(int(hi[i])), L + self.precopy_lead)
                if dst is None:
                    continue
                npg = -(-L // PAGE)
                self.sessions[rid] = [src, dst, npg]
                inflight[src] += 1
                ev.precopies.append((rid, src, dst, npg))
        # 3c. intra-stage rebalancing of overloaded instances via bid-ask
        if self.rebalance_every > 0 and self.step_no % self.rebalance_every == 0:
            self._rebalance(ev, inflight)
        # 4. arrivals: queued first, then one new request per retirement
        pending, self.queue = self.queue, []
        for _ in range(len(done)):
            pending.append(self.stream.next())
        for rid, I, O in pending:
            r = self._place(rid, I, O, I)
            if r is not None:
                ev.admitted.append((rid, r, I))
        return ev

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
        for x in data.ravel().tolist():
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

    def apply(self, ev: StepEvents, comm):
        """Apply one step's events to this rank: retire, grow page lists (new tokens),
        migrate KV pages out/in (P2P), admit new requests."""
        me = self.rank
        for rid, r in ev.retired:
            if r == me and rid in self.pages:
                self.ops.free(self.pool, self._drop(rid))
        # growth: the step's new token opens a new page when L-1 is a multiple of 16
        sim = self.sim
        mig_out = {m[0] for m in ev.migrations if m[1] == me} | {p[0] for p in ev.precopies if p[1] == me}
        grow = np.nonzero(sim.active & ((sim.L - 1) % PAGE == 0))[0]
        for i in grow:
            rid = int(sim.rid[i])
            if rid in self.pages and (int(sim.rank[i]) == me or rid in mig_out):
                need = -(-int(sim.L[i]) // PAGE)
                if need > len(self.pages[rid]):
                    self._append(rid, self.ops.alloc(self.pool, need - len(self.pages[rid])))
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
        nbytes = self.ops.transfer(self.pool, sends, recvs, comm, any_transfer=bool(ev.precopies or ev.migrations))
        for rid, pages in done_in:
            self._add(rid, pages)
        for pages in done_out:
            self.ops.free(self.pool, pages)
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

    def __init__(self, device, slot_bytes: int = 1 << 20, depth: int = 4):
        import torch
        self.torch, self.device, self.slot_bytes, self.depth = torch, device, slot_bytes, depth
        self.h = [torch.empty(slot_bytes, dtype=torch.uint8).pin_memory() for _ in range(depth)]
        self.d = [torch.empty(slot_bytes, dtype=torch.uint8, device=device) for _ in range(depth)]
        self.ev = [None] * depth
        self.i = 0

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
            self.ev[k].synchronize()
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
    KV-page transport (l4_pack_pages -> NCCL send/recv -> l4_unpack_pages)."""

    def __init__(self, shape, device, seed=0):
        import torch
        from . import l4
        self.torch, self.l4, self.shape, self.device = torch, l4, shape, device
        self.seed = seed
        self.h2d = H2DRing(device)

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
        return dict(k=k, v=v, alloc=self.l4.PagePool(num_pages), view=self.l4.kv_view(k, v))

    def alloc(self, pool, n):
        return pool["alloc"].alloc(n).tolist()

    def free(self, pool, pages):
        pool["alloc"].free(pages)

    def make_table(self, slots, max_pages):
        return self.torch.zeros(slots * max_pages, dtype=self.torch.int32, device=self.device)

    def table_update(self, table, pos, val):
        """Scatter this step's page-id deltas into the device block table (pinned H2D, async)."""
        p, v = self.h2d.put(pos, val)
        table.index_copy_(0, p.long(), v)

    # ---------------------------------------------------------------- one-sided (CUDA IPC)
    def setup_ipc(self, pool, rank: int, world: int, group=None):
        """Map every peer's KV pools into this process (CUDA IPC; handles + offsets travel over
        the CPU process group `group`).  Afterwards transfer() pushes pages one-sidedly."""
        import torch.distributed as dist
        l4 = self.l4
        hk, ok = l4.ipc_get_handle(pool["k"].data_ptr())
        hv, ov = l4.ipc_get_handle(pool["v"].data_ptr())
        mine = (hk, ok, hv, ov)
        peers = [None] * world
        dist.all_gather_object(peers, mine, group=group)
        view = pool["view"]
        self.ipc_group, self.ipc_rank, self.ipc_views, self.ipc_bases = group, rank, {}, []
        for r, (pk, pok, pv, pov) in enumerate(peers):
            if r == rank:
                continue
            bk, bv = l4.ipc_open_handle(pk), l4.ipc_open_handle(pv)
            self.ipc_bases += [bk, bv]
            self.ipc_views[r] = l4.kv_view(None, None, device=view.device, num_layers=view.num_layers,
                                           num_pages=view.num_pages, layer_stride_bytes=view.layer_stride_bytes,
                                           page_bytes=view.page_bytes, k_ptr=bk + pok, v_ptr=bv + pov)

    def close_ipc(self):
        for b in getattr(self, "ipc_bases", []):
            self.l4.ipc_close_handle(b)
        self.ipc_bases, self.ipc_views = [], {}

    def _transfer_ipc(self, pool, sends, recvs, any_transfer):
        """One-sided: the receivers' destination page lists (allocated in their idle slots)
        reach the senders over the CPU group; each sender writes its pages straight into the
        receiver's pool (l4_copy_pages over the IPC mapping; NVLink across GPUs), then a
        barrier publishes them.  Every rank takes part whenever any rank transfers."""
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
        for dst, pages in sends:
            dpages = queue[(me, dst)].pop(0)
            assert len(dpages) == len(pages)
            if pages:
                self.l4.copy_pages(pool["view"], pages, self.ipc_views[dst], dpages)
            nbytes += len(pages) * 2 * pb
        nbytes += sum(len(p) for _, p in recvs) * 2 * pb
        self.torch.cuda.current_stream().synchronize()   # the pushes have landed
        dist.barrier(group=self.ipc_group)
        return nbytes

    def transfer(self, pool, sends, recvs, comm, any_transfer=None):
        """sends = [(dst rank, src page ids)], recvs = [(src rank, dst page ids)] in the global
        event order: pack -> batched NCCL P2P -> unpack straight into the receiver's pages
        (allocated by the caller in idle slots), or the one-sided IPC push after
        setup_ipc().  Returns bytes moved by this rank."""
        torch, l4, dist = self.torch, self.l4, comm
        if getattr(self, "ipc_views", None) is not None and hasattr(self, "ipc_rank"):
            return self._transfer_ipc(pool, sends, recvs,
                                      any_transfer if any_transfer is not None else bool(sends or recvs))
        if not sends and not recvs:
            return 0
        pb = pool["view"].page_bytes
        # NCCL moves device buffers over NVLink; the gloo backend (development: several ranks
        # sharing one GPU) needs host buffers, so the staging goes through host memory there.
        host = dist.get_backend() == "gloo"
        ops, bufs, nbytes = [], [], 0
        for dst, pages in sends:
            st = torch.empty(max(len(pages), 1) * 2 * pb, dtype=torch.uint8, device=self.device)
            if pages:
                l4.pack_pages(pool["view"], pages, st)
            ops.append(dist.P2POp(dist.isend, st.cpu() if host else st, dst))
            nbytes += len(pages) * 2 * pb
        for src, pages in recvs:
            st = torch.empty(max(len(pages), 1) * 2 * pb, dtype=torch.uint8, device="cpu" if host else self.device)
            ops.append(dist.P2POp(dist.irecv, st, src))
            bufs.append((pages, st))
            nbytes += len(pages) * 2 * pb
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        for pages, st in bufs:
            if pages:
                l4.unpack_pages(pool["view"], pages, st.to(self.device) if host else st)
        return nbytes
