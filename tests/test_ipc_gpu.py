"""GPU test of the cross-process one-sided migration path (l4_ipc_get_handle / open / close +
l4_migrate into IPC-mapped pools): the receiver process exports its KV pools, the
sender process maps them and pushes a request's pages straight into the receiver's idle pages.
Both processes share cuda:0 here (the development pool has one GPU); across GPUs the same calls
map a peer GPU's memory over NVLink.  The pools are sub-allocations of PyTorch's caching
allocator, so the exported offsets matter."""
import multiprocessing as mp
import os
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LAYERS, PAGES, HKV = 3, 64, 2


def _sender(handles, src_pages, out_q):
    sys.path.insert(0, ROOT)
    import torch as t
    from paper_2512_19179_b200 import l4
    try:
        t.cuda.set_device(0)
        (hk, ok), (hv, ov) = handles
        bk, bv = l4.ipc_open_handle(hk), l4.ipc_open_handle(hv)
        g = t.Generator(device="cuda").manual_seed(7)
        k = t.randn(LAYERS, PAGES, HKV, 16, 128, device="cuda", generator=g).to(t.bfloat16)
        v = t.randn(LAYERS, PAGES, HKV, 16, 128, device="cuda", generator=g).to(t.bfloat16)
        src = l4.kv_view(k, v, num_layers=LAYERS)
        dst = l4.kv_view(None, None, device=0, num_layers=LAYERS, num_pages=PAGES,
                         layer_stride_bytes=src.layer_stride_bytes, page_bytes=src.page_bytes,
                         k_ptr=bk + ok, v_ptr=bv + ov)
        pool = l4.PagePool(PAGES)
        pool.alloc(5)                                  # the receiver's pages 0..4 are in use
        dst_pages = l4.migrate(src, src_pages, dst, pool)
        t.cuda.synchronize()
        l4.ipc_close_handle(bk)
        l4.ipc_close_handle(bv)
        out_q.put(("ok", dst_pages.tolist(), k[:, src_pages].view(t.int16).cpu().numpy(),
                   v[:, src_pages].view(t.int16).cpu().numpy()))
    except Exception as e:  # noqa: BLE001 - reported to the parent
        out_q.put(("error", repr(e), None, None))


def test_migrate_into_ipc_mapped_pools():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    sys.path.insert(0, ROOT)
    from paper_2512_19179_b200 import l4
    torch.cuda.set_device(0)
    pad = torch.empty(12345, dtype=torch.uint8, device="cuda")   # make the pools sub-allocations
    k = torch.zeros(LAYERS, PAGES, HKV, 16, 128, device="cuda", dtype=torch.bfloat16)
    v = torch.zeros_like(k)
    torch.cuda.synchronize()
    handles = (l4.ipc_get_handle(k.data_ptr()), l4.ipc_get_handle(v.data_ptr()))
    src_pages = [9, 3, 40, 41, 17]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_sender, args=(handles, src_pages, q))
    p.start()
    status, dst_pages, ek, ev = q.get(timeout=300)
    p.join(timeout=60)
    assert status == "ok", dst_pages
    assert dst_pages == [5, 6, 7, 8, 9]                # lowest idle pages of the receiver (Z27)
    torch.cuda.synchronize()
    got_k = k[:, dst_pages].view(torch.int16).cpu().numpy()
    got_v = v[:, dst_pages].view(torch.int16).cpu().numpy()
    assert np.array_equal(got_k, ek) and np.array_equal(got_v, ev)
    untouched = [i for i in range(PAGES) if i not in dst_pages]
    assert not k[:, untouched].any() and not v[:, untouched].any()
    del pad
