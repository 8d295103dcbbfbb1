"""GPU tests of KV-page migration (loopback on one GPU: src and dst pools on the
same device use the same copy kernel as a peer / IPC destination)."""
import numpy as np
import pytest
import torch

import synth
from oracle import pool as opool
from paper_2512_19179_b200 import l4

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _pools(num_pages, layers=3, Hkv=2, seed=0):
    g = torch.Generator(device="cuda").manual_seed(seed)
    k = torch.randn(layers, num_pages, Hkv, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(layers, num_pages, Hkv, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
    return k, v


def test_migrate_loopback_bytes_and_allocator():
    src_k, src_v = _pools(50, seed=1)
    dst_k = torch.zeros(3, 40, 2, 16, 128, dtype=torch.bfloat16, device="cuda")
    dst_v = torch.zeros_like(dst_k)
    src = l4.kv_view(src_k, src_v, num_layers=3)
    dst = l4.kv_view(dst_k, dst_v, num_layers=3)
    pool = l4.PagePool(40)
    ref_pool = opool.PagePool(40)
    busy = pool.alloc(5)
    ref_pool.alloc(5)
    src_pages = [17, 3, 44, 9, 0, 31]
    dpages = l4.migrate(src, src_pages, dst, pool)
    torch.cuda.synchronize()
    assert dpages.tolist() == ref_pool.alloc(len(src_pages)) == [5, 6, 7, 8, 9, 10]
    for s, d in zip(src_pages, dpages):
        assert torch.equal(dst_k[:, d], src_k[:, s]) and torch.equal(dst_v[:, d], src_v[:, s])
    # untouched pages stay zero
    assert int(dst_k[:, 11:].abs().sum().item()) == 0
    # no idle cache -> NO_PAGES, nothing copied, pool unchanged (Z28)
    before = pool.num_free()
    with pytest.raises(l4.NoPagesError):
        l4.migrate(src, list(range(50)), dst, pool)
    assert pool.num_free() == before
    pool.free(busy)


def test_migrate_large_request_multi_launch():
    """More pages than one launch carries (1024) and an event for completion."""
    src_k, src_v = _pools(3000, layers=2, Hkv=1, seed=2)
    dst_k = torch.zeros(2, 3000, 1, 16, 128, dtype=torch.bfloat16, device="cuda")
    dst_v = torch.zeros_like(dst_k)
    src = l4.kv_view(src_k, src_v, num_layers=2)
    dst = l4.kv_view(dst_k, dst_v, num_layers=2)
    pool = l4.PagePool(3000)
    sp = np.random.default_rng(0).permutation(3000)[:2500]
    ev = torch.cuda.Event()
    dp = l4.migrate(src, sp, dst, pool, done_event=ev)
    ev.synchronize()
    idx_s = torch.as_tensor(sp, device="cuda", dtype=torch.long)
    idx_d = torch.as_tensor(dp, device="cuda", dtype=torch.long)
    assert torch.equal(dst_k[:, idx_d], src_k[:, idx_s]) and torch.equal(dst_v[:, idx_d], src_v[:, idx_s])


def test_pack_unpack_roundtrip():
    src_k, src_v = _pools(20, seed=3)
    src = l4.kv_view(src_k, src_v, num_layers=3)
    pages = [4, 19, 0, 7]
    pb = src.page_bytes
    staging = torch.empty(len(pages) * 3 * 2 * pb, dtype=torch.uint8, device="cuda")
    l4.pack_pages(src, pages, staging)
    dst_k = torch.zeros_like(src_k)
    dst_v = torch.zeros_like(src_v)
    dst = l4.kv_view(dst_k, dst_v, num_layers=3)
    dpages = [1, 2, 3, 5]
    l4.unpack_pages(dst, dpages, staging)
    torch.cuda.synchronize()
    for s, d in zip(pages, dpages):
        assert torch.equal(dst_k[:, d], src_k[:, s]) and torch.equal(dst_v[:, d], src_v[:, s])
    # staging order: [page][layer][K, V]
    st = staging.view(len(pages), 3, 2, -1)
    assert torch.equal(st[1, 2, 1], src_v[2, 19].reshape(-1).view(torch.uint8))


def test_attention_identical_after_migration():
    """Attention on the destination after migration is bit-identical to the source."""
    shape = synth.AttnShape("t", 32, 8)
    table = synth.make_page_table([700, 33, 4096], seed=1, spare_pages=10)
    q, k, v = synth.make_qkv_cpu(shape, table, seed=1)
    q, k, v = q.cuda(), k.cuda(), v.cuda()
    ip = torch.from_numpy(table.indptr).cuda()
    ix = torch.from_numpy(table.indices).cuda()
    kl = torch.from_numpy(table.kv_len).cuda()
    out_src, lse_src = l4.decode_attention(q, k, v, ip, ix, kl)
    dst_k = torch.full((table.total_pages + 7, 8, 16, 128), float("nan"), dtype=torch.bfloat16, device="cuda")
    dst_v = torch.full_like(dst_k, float("nan"))
    pool = l4.PagePool(dst_k.shape[0])
    pool.alloc(7)
    src = l4.kv_view(k, v)
    dst = l4.kv_view(dst_k, dst_v)
    new_indices = []
    for b in range(table.batch):
        pages = table.indices[table.indptr[b]:table.indptr[b + 1]]
        new_indices.extend(l4.migrate(src, pages, dst, pool).tolist())
    ix2 = torch.tensor(new_indices, dtype=torch.int32, device="cuda")
    out_dst, lse_dst = l4.decode_attention(q, dst_k, dst_v, ip, ix2, kl)
    torch.cuda.synchronize()
    assert torch.equal(out_src, out_dst) and torch.equal(lse_src, lse_dst)
