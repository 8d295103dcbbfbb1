"""GPU test of the pipeline's one-sided page transport (DeviceOps.setup_ipc: every rank maps its
peers' KV pools through CUDA IPC and the sender writes a migrating request's pages straight into
the receiver's idle pages).  Two rank processes share cuda:0 (the development pool has
one GPU), the control plane is replicated as in bench.py, metadata and barriers go over gloo.
Every page is tagged with its owner; after each step every migrated-in page must carry its
request's tag in K and V, and page accounting must be conserved on every rank."""
import os
import socket
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _tag(rid):  # small integers are exact in bf16
    return float(rid % 97 + 1)


def _worker(rank, world, port, steps, lead, out_q):
    sys.path.insert(0, ROOT)
    import torch as t
    import torch.distributed as dist
    import synth
    from paper_2512_19179_b200 import pipeline
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t.cuda.set_device(0)
        stages = [(0, 1500, 1), (1500, 262144, world - 1)]
        sim = pipeline.ClusterSim(stages, concurrency=48 * world, seed=5, token_budget=400_000, batch_cap=256,
                                  precopy_lead=lead)
        shape = synth.AttnShape("ipc", 4, 2)
        rt = pipeline.RankRuntime(sim, rank, 400_000 // 16 * 2, shape, pipeline.DeviceOps(shape, "cuda:0", rank))
        rt.ops.setup_ipc(rt.pool, rank, world)
        pool = rt.pool

        def tag(rid, pages):
            idx = t.tensor(pages, device="cuda", dtype=t.long)
            pool["k"][idx] = _tag(rid)
            pool["v"][idx] = -_tag(rid)

        for rid, pages in rt.pages.items():
            tag(rid, pages)
        t.cuda.synchronize()
        dist.barrier()
        checked = 0
        for _ in range(steps):
            before = {rid: len(p) for rid, p in rt.pages.items()}
            ev = sim.step()
            rt.apply(ev, dist)
            rt.ops.before_decode()   # this stream waits for the senders' pushes (their IPC events)
            migrated_in = {m[0] for m in ev.migrations if m[2] == rank}
            for rid, pages in rt.pages.items():
                if rid in migrated_in:
                    idx = t.tensor(pages, device="cuda", dtype=t.long)
                    assert bool((pool["k"][idx] == _tag(rid)).all()), f"K pages of {rid} on rank {rank}"
                    assert bool((pool["v"][idx] == -_tag(rid)).all()), f"V pages of {rid} on rank {rank}"
                    checked += 1
                else:
                    new = pages[before.get(rid, 0):]
                    if new:
                        tag(rid, new)
            t.cuda.synchronize()
            dist.barrier()   # tags written before any peer pushes these pages on
            used = sum(len(p) for p in rt.pages.values()) + sum(len(p) for p in rt.incoming.values())
            pending = sum(len(p) for _, p in pool["pending"])   # freed, waiting for their last reader
            assert pool["alloc"].num_free() + pending == pool["alloc"].num_pages - used, "page accounting"
        fps = [None] * world
        dist.all_gather_object(fps, sim.fingerprint())
        rt.ops.close_ipc()
        out_q.put((rank, len(set(fps)) == 1, checked, dict(rt.stats), None))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        out_q.put((rank, False, 0, {}, repr(e)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,lead", [(2, 0), (3, 4)])
def test_pipeline_ipc_transport(world, lead):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 120, lead, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    errs = [e for *_, e in res if e]
    assert not errs, errs
    assert all(ok for _, ok, _, _, _ in res)
    checked = sum(c for _, _, c, _, _ in res)
    assert checked > 0
    outs = sum(s["migrations_out"] for *_, s, _ in res)
    ins = sum(s["migrations_in"] for *_, s, _ in res)
    assert outs == ins == checked
