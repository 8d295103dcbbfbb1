"""GPU parity tests: l4_decode_attention (CUDA, sm_100a, through the C ABI) vs
the FP64 oracle on the same seeded inputs.  Tolerance: max abs error 2e-3 on
fp32 outputs (BASELINE.json north star); LSE within 2e-3 as well.
"""
import math

import numpy as np
import pytest
import torch

import synth
from oracle import attention as oa
from paper_2512_19179_b200 import l4

pytestmark = pytest.mark.gpu

TOL = 2e-3


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    torch.cuda.init()


def _to_dev(table, q, k, v):
    d = "cuda"
    return (q.to(d), k.to(d), v.to(d), torch.from_numpy(table.indptr).to(d), torch.from_numpy(table.indices).to(d),
            torch.from_numpy(table.kv_len).to(d))


def _run_gpu(table, q, k, v, **kw):
    qd, kd, vd, ip, ix, kl = _to_dev(table, q, k, v)
    out, lse = l4.decode_attention(qd, kd, vd, ip, ix, kl, **kw)
    torch.cuda.synchronize()
    return out.double().cpu().numpy(), lse.double().cpu().numpy()


def _check(out, lse, ref_out, ref_lse, tol=TOL):
    err = np.max(np.abs(out - ref_out)) if out.size else 0.0
    assert err <= tol, f"max abs err {err}"
    fin = np.isfinite(ref_lse)
    assert np.all(np.isneginf(lse[~fin]))
    if fin.any():
        lerr = np.max(np.abs(lse[fin] - ref_lse[fin]))
        assert lerr <= tol, f"lse err {lerr}"
    return err


def _case(lens, Hq, Hkv, seed=0, q_scale=1.0, spare=3, layout="fragmented"):
    shape = synth.AttnShape("t", Hq, Hkv)
    table = synth.make_page_table(np.asarray(lens), seed=seed, spare_pages=spare, layout=layout)
    q, k, v = synth.make_qkv_cpu(shape, table, seed=seed, q_scale=q_scale, poison_unused=True)
    ref_out, ref_lse = oa.paged_decode_attention(q, k, v, table.indptr, table.indices, table.kv_len, Hkv)
    return shape, table, q, k, v, ref_out, ref_lse


def test_c1_config():
    """BASELINE.json configs[0]: 8 q / 2 kv heads, B=4, L = {16, 64, 256, 1024}."""
    shape, table, q, k, v, ro, rl = _case(synth.lengths_c1(), 8, 2)
    out, lse = _run_gpu(table, q, k, v)
    err = _check(out, lse, ro, rl)
    assert err < 1e-4


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("chunk", [0, -1, 1, 3])
def test_random_shapes(G, chunk):
    rng = np.random.default_rng(100 + G * 10 + chunk)
    lens = [0, 1, 15, 16, 17, 31, 33, 100, 255, 256, 257, 1000] + rng.integers(1, 3000, size=6).tolist()
    Hkv = 2 if G == 8 else 3
    shape, table, q, k, v, ro, rl = _case(lens, Hkv * G, Hkv, seed=G)
    out, lse = _run_gpu(table, q, k, v, chunk_pages=chunk)
    _check(out, lse, ro, rl)


def test_peaked_softmax():
    """q x 4 makes the softmax peaked (adversarial for the probability precision, Z23)."""
    shape, table, q, k, v, ro, rl = _case([16, 64, 256, 1024, 3000], 32, 8, seed=5, q_scale=4.0)
    for chunk in (0, 2):
        out, lse = _run_gpu(table, q, k, v, chunk_pages=chunk)
        _check(out, lse, ro, rl)


def test_bf16_output():
    shape, table, q, k, v, ro, rl = _case([5, 77, 400, 2048], 16, 4, seed=9)
    out, lse = _run_gpu(table, q, k, v, out_dtype=l4.L4_DT_BF16)
    # bf16 rounding of the output adds up to 2^-9 relative (Z22)
    assert np.max(np.abs(out - ro) - np.abs(ro) * 2.0 ** -8) <= TOL
    _check(out * 0, lse, ro * 0, rl)


def test_split_invariance_and_repeat_runs():
    """Unsplit vs split at several chunk sizes agree; repeated runs with one plan are bit-identical."""
    shape, table, q, k, v, ro, rl = _case([1, 40, 700, 5000], 32, 8, seed=3)
    base, base_lse = _run_gpu(table, q, k, v, chunk_pages=-1)
    for chunk in (1, 2, 7, 64):
        out, lse = _run_gpu(table, q, k, v, chunk_pages=chunk)
        assert np.max(np.abs(out - base)) < 2e-5
        assert np.max(np.abs(lse - base_lse)[np.isfinite(base_lse)]) < 2e-5
    qd, kd, vd, ip, ix, kl = _to_dev(table, q, k, v)
    params = l4.make_params(table.batch, 32, 8, chunk_pages=2)
    ws = l4.alloc_workspace(params, table.total_pages)
    l4.decode_plan(params, kl, ip, table.total_pages, ws)
    outs = []
    for _ in range(3):
        o = torch.empty(table.batch, 32, 128, device="cuda")
        lz = torch.empty(table.batch, 32, device="cuda")
        l4.decode_run(params, qd, kd, vd, ix, o, lz, ws)
        outs.append((o.cpu(), lz.cpu()))
    torch.cuda.synchronize()
    for o, lz in outs[1:]:
        assert torch.equal(o, outs[0][0]) and torch.equal(lz, outs[0][1])


def test_page_layout_independence_bitwise():
    lens = [16, 100, 513, 2000]
    shape, t1, q, k, v, ro, rl = _case(lens, 16, 4, seed=4, layout="contiguous", spare=0)
    out1, lse1 = _run_gpu(t1, q, k, v)
    perm = np.random.default_rng(1).permutation(t1.num_pages)
    k2 = torch.empty_like(k)
    v2 = torch.empty_like(v)
    k2[torch.as_tensor(perm)] = k
    v2[torch.as_tensor(perm)] = v
    t2 = synth.PageTable(kv_len=t1.kv_len, indptr=t1.indptr, indices=perm[t1.indices].astype(np.int32),
                         num_pages=t1.num_pages)
    out2, lse2 = _run_gpu(t2, q, k2, v2)
    assert np.array_equal(out1, out2) and np.array_equal(lse1, lse2)


def test_plan_covers_every_token_once():
    rng = np.random.default_rng(11)
    lens = np.concatenate([[0, 1, 16, 17], rng.integers(1, 20000, size=60), [131072]])
    table = synth.make_page_table(lens, seed=0)
    kl = torch.from_numpy(table.kv_len).cuda()
    ip = torch.from_numpy(table.indptr).cuda()
    for chunk in (0, 5):
        params = l4.make_params(table.batch, 32, 8, chunk_pages=chunk)
        ws = l4.alloc_workspace(params, table.total_pages)
        l4.decode_plan(params, kl, ip, table.total_pages, ws)
        items = l4.plan_items(ws)
        info = l4.plan_info(ws)
        assert info.num_items == len(items)
        covered = {}
        sizes = []
        for b, h, pb, pe, last_valid, part_base, ns, s in items.tolist():
            L = int(table.kv_len[b])
            base = int(table.indptr[b])
            npg = (L + 15) // 16
            assert base <= pb <= pe <= base + npg
            if L > 0:
                assert pe > pb
            for p in range(pb, pe):
                key = (b, h, p)
                assert key not in covered
                covered[key] = 1
            if pe == base + npg and L > 0:
                assert last_valid == L - (npg - 1) * 16
            # ordering key = bit_length of the request's largest split under the plain chunk C
            C = info.chunk_pages
            plain_ns = 1 if npg <= 2 * C else -(-npg // C)
            sizes.append(0 if npg == 0 else -(-npg // plain_ns))
            if plain_ns > 1:  # the quad-bin bound: a split request's largest split exceeds 2C/3
                assert 3 * sizes[-1] > 2 * C
            # only the guided tail (automatic chunk) splits differently: split requests whose work
            # starts in the plan's tail get pieces of the tail chunk (at most 512)
            if ns != plain_ns:
                Ct = info.tail_chunk_pages
                assert chunk == 0 and Ct > 0 and plain_ns > 1 and ns == min(512, -(-npg // Ct)) and ns > plain_ns
        expect = sum(8 * ((int(L) + 15) // 16) for L in table.kv_len)
        assert len(covered) == expect
        # length-binned, longest bin first: bins are non-increasing along the work list
        bl = [int(x).bit_length() for x in sizes]
        assert all(a >= b for a, b in zip(bl, bl[1:]))


def test_single_bin_fast_path_plan_equals_general_plan():
    """The planner's fast path (no split request, every request in one length bin: the stable
    LPT order is the request order) builds the same work list as the general counting-sort path:
    the same batch plus one shorter request (a second, lower bin, ranked last) takes the general
    path, and its work list must start with the fast path's, item for item."""
    rng = np.random.default_rng(21)
    lens_a = rng.integers(500, 1000, size=300)            # 32..63 pages: one bin (bit_length 6)
    lens_b = np.concatenate([lens_a, [5]])                 # + one 1-page request (bin 1)
    plans = []
    for lens in (lens_a, lens_b):
        table = synth.make_page_table(lens, seed=0)
        params = l4.make_params(table.batch, 32, 8)
        ws = l4.alloc_workspace(params, table.total_pages)
        l4.decode_plan(params, torch.from_numpy(table.kv_len).cuda(), torch.from_numpy(table.indptr).cuda(),
                       table.total_pages, ws)
        plans.append((l4.plan_info(ws), l4.plan_items(ws)))
    (ia, pa), (ib, pb) = plans
    assert ia.chunk_pages == ib.chunk_pages and ia.max_splits == ib.max_splits == 1
    assert len(pa) == 300 * 8 and len(pb) == 301 * 8
    np.testing.assert_array_equal(pa, pb[: len(pa)])
    assert pb[-8:, 0].tolist() == [300] * 8                  # the short request comes last
    assert pa[:, 0].tolist() == np.repeat(np.arange(300), 8).tolist()  # request order, heads ascending
    assert pa[:, 1].tolist() == np.tile(np.arange(8), 300).tolist()


def test_empty_batch_and_all_empty_requests():
    shape, table, q, k, v, ro, rl = _case([0, 0, 0], 8, 2)
    out, lse = _run_gpu(table, q, k, v)
    assert np.all(out == 0) and np.all(np.isneginf(lse))
    params = l4.make_params(0, 8, 2)
    assert l4.lib().l4_decode_plan(params, None, None, 0, None, 0, None) == 0


def _poison_unread(k, v, table):
    """NaN into every slot no request reads (tails of last pages, pages outside the table), on the
    device (vectorised form of synth.poison_unread_slots for full-size pools)."""
    npg = np.diff(table.indptr.astype(np.int64))
    used = np.zeros(table.num_pages, dtype=bool)
    used[table.indices] = True
    tail = np.ones((table.num_pages, 16), dtype=bool)
    tail[used] = False
    last = table.indices[table.indptr[1:][npg > 0] - 1]
    lv = table.kv_len[npg > 0] - (npg[npg > 0] - 1) * 16
    for t in range(1, 16):
        tail[last[lv <= t], t] = True
    m = torch.from_numpy(tail).cuda()[:, None, :, None]
    k.masked_fill_(m, float("nan"))
    v.masked_fill_(m, float("nan"))


def _full_size(lens, shape, seed):
    """Full-size parity in the bench launch configuration (auto plan, single launch, back to back,
    plain and early-input calls): EVERY output row of a plain call against the FP64 oracle, with
    unread KV slots NaN-poisoned; the split partials NaN-poisoned before the repeated calls, which
    must be bitwise identical to the first call."""
    table = synth.make_page_table(lens, seed=seed, spare_pages=64)
    g = torch.Generator(device="cuda").manual_seed(seed)
    B = table.batch
    q = torch.randn(B, shape.num_q_heads, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
    _poison_unread(k, v, table)
    ip = torch.from_numpy(table.indptr).cuda()
    ix = torch.from_numpy(table.indices).cuda()
    kl = torch.from_numpy(table.kv_len).cuda()
    out, lse = l4.decode_attention(q, k, v, ip, ix, kl)
    torch.cuda.synchronize()
    for flags in (0, l4.L4_DECODE_EARLY_PLAN, l4.L4_DECODE_EARLY_INPUTS):
        params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads, flags=flags)
        ws = l4.alloc_workspace(params, table.total_pages)
        l4.poison_partials(params, ws)
        o2, l2 = torch.empty_like(out), torch.empty_like(lse)
        for _ in range(3):
            l4.attention_call(params, q, k, v, ip, ix, kl, table.total_pages, o2, l2, ws)
            torch.cuda.synchronize()
            assert torch.equal(o2, out) and torch.equal(l2, lse)
    ro, rl = oa.paged_decode_attention(q, k, v, table.indptr, table.indices, table.kv_len, shape.num_kv_heads)
    return _check(out.double().cpu().numpy(), lse.double().cpu().numpy(), ro, rl)


def test_full_size_short_stage():
    """bench.py's stage-shaped [0, 1024) batch (B = 1024 at the Llama-3-8B shape, the short
    stage an L4 instance serves): quad units at full size, ragged lengths around the bench's 530."""
    lens = np.random.default_rng(530).integers(300, 761, size=1024)
    lens[0], lens[-1] = 1, 1023
    _full_size(lens, synth.SHAPE_LLAMA3_8B, 0)


def test_full_size_short_stage_70b():
    """B = 1024 short requests at the Llama-3-70B shape (G = 8 quad units, Q rows through the ring)."""
    lens = np.random.default_rng(64).integers(1, 400, size=1024)
    _full_size(lens, synth.SHAPE_LLAMA3_70B, 1)


def test_full_size_c2():
    _full_size(synth.lengths_c2(), synth.SHAPE_LLAMA3_8B, 0)


def test_full_size_c3():
    _full_size(synth.lengths_c3(0), synth.SHAPE_LLAMA3_8B, 0)


def test_full_size_fig2_mixed():
    """Fig. 2 (`fig:interference`) analogue at full size: batch 512, 32 requests of 50,000 tokens
    among 1,000-token ones — long split requests and many short unsplit ones in one launch."""
    _full_size(synth.lengths_fig2(512, 32, 1000, 50000), synth.SHAPE_LLAMA3_8B, 3)


def test_full_size_long_stage():
    """A long-stage batch (12 requests around 84K tokens, C3's [64K, 128K) class refilled):
    every request split tens of ways, two-level combines."""
    lens = np.random.default_rng(12).integers(70000, 100001, size=12)
    _full_size(lens, synth.SHAPE_LLAMA3_8B, 4)


def test_full_size_c4():
    _full_size(synth.lengths_c4(0), synth.SHAPE_LLAMA3_70B, 0)


def test_repeat_calls_bitwise_c4_many():
    """The split-combine repeat check that exposed the missing proxy fence: 200
    back-to-back C4 calls (early inputs, the flaky configuration) bitwise equal to the first."""
    shape, lens = synth.SHAPE_LLAMA3_70B, synth.lengths_c4(0)
    table = synth.make_page_table(lens, seed=0, spare_pages=64)
    g = torch.Generator(device="cuda").manual_seed(0)
    B = table.batch
    q = torch.randn(B, shape.num_q_heads, 128, device="cuda", generator=g).to(torch.bfloat16)
    k = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
    v = torch.randn(table.num_pages, shape.num_kv_heads, 16, 128, device="cuda", generator=g).to(torch.bfloat16)
    ip, ix, kl = (torch.from_numpy(x).cuda() for x in (table.indptr, table.indices, table.kv_len))
    out, lse = l4.decode_attention(q, k, v, ip, ix, kl)
    params = l4.make_params(B, shape.num_q_heads, shape.num_kv_heads, flags=l4.L4_DECODE_EARLY_INPUTS)
    ws = l4.alloc_workspace(params, table.total_pages)
    outs = [torch.empty_like(out) for _ in range(8)]
    lses = [torch.empty_like(lse) for _ in range(8)]
    bad = 0
    for rep in range(25):
        for i in range(8):
            l4.attention_call(params, q, k, v, ip, ix, kl, table.total_pages, outs[i], lses[i], ws)
        torch.cuda.synchronize()
        bad += sum(int(not (torch.equal(o, out) and torch.equal(z, lse))) for o, z in zip(outs, lses))
    assert bad == 0


# ----------------------------------------------------------------------------- fused single-launch path
def _dev_case(lens, Hq, Hkv, seed):
    shape, table, q, k, v, ro, rl = _case(lens, Hq, Hkv, seed=seed)
    return (table, ro, rl) + _to_dev(table, q, k, v)


def _plan_run(params, table, qd, kd, vd, ip, ix, kl, ws):
    o = torch.full((table.batch, params.num_q_heads, 128), float("nan"), device="cuda")
    lz = torch.full((table.batch, params.num_q_heads), float("nan"), device="cuda")
    l4.decode_plan(params, kl, ip, table.total_pages, ws)
    l4.decode_run(params, qd, kd, vd, ix, o, lz, ws)
    return o, lz


def _fused(params, table, qd, kd, vd, ip, ix, kl, ws):
    # NaN-filled outputs: a work item the kernel's unit mapping skipped leaves NaN rows behind
    o = torch.full((table.batch, params.num_q_heads, 128), float("nan"), device="cuda")
    lz = torch.full((table.batch, params.num_q_heads), float("nan"), device="cuda")
    l4.attention_call(params, qd, kd, vd, ip, ix, kl, table.total_pages, o, lz, ws)
    return o, lz


@pytest.mark.parametrize("G", [1, 2, 4, 8])
@pytest.mark.parametrize("chunk", [0, 2, -1])
def test_fused_equals_plan_plus_run_bitwise(G, chunk):
    """l4_decode_attention (one launch, per-CTA shared-memory plan) builds the same work list as
    plan_kernel: outputs are bit-identical to l4_decode_plan + l4_decode_run, and match the oracle."""
    rng = np.random.default_rng(7 * G + chunk)
    lens = [0, 1, 16, 17, 255, 4000] + rng.integers(1, 2500, size=40).tolist() + [0]
    Hkv = 2
    table, ro, rl, qd, kd, vd, ip, ix, kl = _dev_case(lens, Hkv * G, Hkv, seed=G)
    params = l4.make_params(table.batch, Hkv * G, Hkv, chunk_pages=chunk)
    ws = l4.alloc_workspace(params, table.total_pages)
    o1, l1 = _plan_run(params, table, qd, kd, vd, ip, ix, kl, ws)
    o2, l2 = _fused(params, table, qd, kd, vd, ip, ix, kl, ws)
    o3, l3 = _fused(params, table, qd, kd, vd, ip, ix, kl, ws)   # repeat: self-cleaning state
    pe = l4.make_params(table.batch, Hkv * G, Hkv, chunk_pages=chunk, flags=l4.L4_DECODE_EARLY_INPUTS)
    early = [_fused(pe, table, qd, kd, vd, ip, ix, kl, ws) for _ in range(3)]  # back to back (PDL overlap)
    pp = l4.make_params(table.batch, Hkv * G, Hkv, chunk_pages=chunk, flags=l4.L4_DECODE_EARLY_PLAN)
    eplan = [_fused(pp, table, qd, kd, vd, ip, ix, kl, ws) for _ in range(3)]  # plan under the previous tail
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    assert torch.equal(o2, o3) and torch.equal(l2, l3)
    for o4, l4_ in early + eplan:
        assert torch.equal(o2, o4) and torch.equal(l2, l4_)
    _check(o2.double().cpu().numpy(), l2.double().cpu().numpy(), ro, rl)


@pytest.mark.parametrize("G,chunk", [(1, 0), (2, 0), (4, 0), (8, 0), (4, -1), (4, 3), (8, 6)])
def test_quad_units_short_batch(G, chunk):
    """Large batches of short requests run as quad units (four unsplit items per CTA unit, one
    per consumer warp, no merge), with the long requests CTA-wide before them and a CTA-wide
    tail after them.  8192 items (B = 1024, 8 kv heads) clear the >= 4 quads per CTA threshold.
    Ragged lengths (NaN-poisoned tails), empty requests, items of 32..63 pages (the second
    block of page ids), fp32 and bf16 outputs; fused == plan + run bitwise; early-input
    back-to-back calls bitwise; oracle within 2e-3.  Forced chunks: -1 (no splits: every item
    of <= 63 pages is quad-eligible), 3 and 6 (quad bins shrink to items of <= 2C/3 pages, the
    split requests' pieces run CTA-wide)."""
    rng = np.random.default_rng(300 + G)
    lens = rng.integers(1, 1009, size=1024)
    lens[:6] = [0, 1, 16, 1008, 513, 0]
    lens[-3:] = [9000, 20000, 3000]  # CTA-wide items ahead of the quad suffix
    Hkv = 8
    table, ro, rl, qd, kd, vd, ip, ix, kl = _dev_case(lens, Hkv * G, Hkv, seed=G)
    params = l4.make_params(table.batch, Hkv * G, Hkv, chunk_pages=chunk)
    ws = l4.alloc_workspace(params, table.total_pages)
    o1, l1 = _plan_run(params, table, qd, kd, vd, ip, ix, kl, ws)
    o2, l2 = _fused(params, table, qd, kd, vd, ip, ix, kl, ws)
    pe = l4.make_params(table.batch, Hkv * G, Hkv, chunk_pages=chunk, flags=l4.L4_DECODE_EARLY_INPUTS)
    early = [_fused(pe, table, qd, kd, vd, ip, ix, kl, ws) for _ in range(3)]
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for o4, l4_ in early:
        assert torch.equal(o2, o4) and torch.equal(l2, l4_)
    _check(o2.double().cpu().numpy(), l2.double().cpu().numpy(), ro, rl)
    pb = l4.make_params(table.batch, Hkv * G, Hkv, out_dtype=l4.L4_DT_BF16, chunk_pages=chunk)
    ob = torch.empty(table.batch, Hkv * G, 128, device="cuda", dtype=torch.bfloat16)
    lb = torch.empty(table.batch, Hkv * G, device="cuda")
    l4.attention_call(pb, qd, kd, vd, ip, ix, kl, table.total_pages, ob, lb, ws)
    torch.cuda.synchronize()
    # bf16 output = the fp32 result rounded once
    assert torch.equal(ob, o2.to(torch.bfloat16))
    assert torch.equal(lb, l2)


@pytest.mark.parametrize("G", [4, 8])
def test_quad_units_few_per_cta(G):
    """The late round-2 quad admission rule (clamp(pages / 10, 1, 4) units per CTA): B = 256
    requests of ~200 tokens give 512 quad units, ~1.7 per CTA, so most CTAs run one or two quads
    and the launch ends on them.  Ragged lengths with NaN-poisoned tails, fused == plan + run
    bitwise, repeated calls bitwise, oracle within 2e-3."""
    rng = np.random.default_rng(500 + G)
    lens = rng.integers(150, 209, size=256)
    lens[:3] = [0, 1, 208]
    Hkv = 8
    table, ro, rl, qd, kd, vd, ip, ix, kl = _dev_case(lens, Hkv * G, Hkv, seed=G)
    params = l4.make_params(table.batch, Hkv * G, Hkv)
    ws = l4.alloc_workspace(params, table.total_pages)
    o1, l1 = _plan_run(params, table, qd, kd, vd, ip, ix, kl, ws)
    o2, l2 = _fused(params, table, qd, kd, vd, ip, ix, kl, ws)
    again = [_fused(params, table, qd, kd, vd, ip, ix, kl, ws) for _ in range(3)]
    torch.cuda.synchronize()
    assert torch.equal(o1, o2) and torch.equal(l1, l2)
    for o3, l3 in again:
        assert torch.equal(o2, o3) and torch.equal(l2, l3)
    _check(o2.double().cpu().numpy(), l2.double().cpu().numpy(), ro, rl)


@pytest.mark.parametrize("Hq", [32, 64])
def test_quad_units_materialised_plan(Hq):
    """B > 1024 takes the materialised plan (planner kernel + run kernel): quad units there too,
    for G = 4 (Q rows in the unit slot) and G = 8 (Q rows through the page ring), vs the oracle."""
    rng = np.random.default_rng(77 + Hq)
    lens = rng.integers(0, 300, size=2048)
    lens[:2] = [4000, 1]
    table, ro, rl, qd, kd, vd, ip, ix, kl = _dev_case(lens, Hq, 8, seed=Hq)
    out, lse = l4.decode_attention(qd, kd, vd, ip, ix, kl)
    torch.cuda.synchronize()
    _check(out.double().cpu().numpy(), lse.double().cpu().numpy(), ro, rl)


def test_fused_workspace_reuse_across_batch_sizes():
    """One workspace, calls with different B (and split-heavy plans) back to back: the split
    counters live in a region independent of B, so no call sees another call's stale items."""
    p_max = l4.make_params(1024, 32, 8)
    ws = None
    for i, (B, hi) in enumerate([(3, 20000), (700, 3000), (5, 60000), (1024, 600), (1, 131072), (40, 9000)]):
        rng = np.random.default_rng(50 + i)
        lens = rng.integers(1, hi, size=B)
        table, ro, rl, qd, kd, vd, ip, ix, kl = _dev_case(lens, 32, 8, seed=i)
        if ws is None:
            ws = l4.alloc_workspace(p_max, 200000)
        params = l4.make_params(B, 32, 8)
        if i % 2:
            o, lz = _plan_run(params, table, qd, kd, vd, ip, ix, kl, ws)
        else:
            o, lz = _fused(params, table, qd, kd, vd, ip, ix, kl, ws)
        torch.cuda.synchronize()
        _check(o.double().cpu().numpy(), lz.double().cpu().numpy(), ro, rl)


def test_fused_batch_limit_and_max_batch():
    """B = 1024 (largest fused batch) and B = 8192 (largest batch, planner-kernel path) vs the oracle."""
    for B, seed in ((1024, 1), (1025, 2), (8192, 3)):
        rng = np.random.default_rng(seed)
        lens = rng.integers(0, 40, size=B)
        lens[rng.integers(0, B, size=4)] = [3000, 1, 0, 777]
        table, ro, rl, qd, kd, vd, ip, ix, kl = _dev_case(lens, 8, 2, seed=seed)
        out, lse = l4.decode_attention(qd, kd, vd, ip, ix, kl)
        torch.cuda.synchronize()
        _check(out.double().cpu().numpy(), lse.double().cpu().numpy(), ro, rl)


def test_longest_request_split_cap():
    """One 2^18-token request (16,384 pages) next to short ones: the split count is capped at
    512 per (request, kv head), so the chunk grows past the automatic choice (8 -> 32 pages)."""
    lens = [1 << 18, 3, 100]
    table, ro, rl, qd, kd, vd, ip, ix, kl = _dev_case(lens, 8, 1, seed=11)
    for chunk in (0, 1):
        out, lse = l4.decode_attention(qd, kd, vd, ip, ix, kl, chunk_pages=chunk)
        torch.cuda.synchronize()
        _check(out.double().cpu().numpy(), lse.double().cpu().numpy(), ro, rl)


@pytest.mark.parametrize("G", [1, 2, 8])
def test_two_level_combine_group_boundaries(G):
    """chunk_pages=1 splits a request of p > 2 pages p ways: split counts around the 16-split
    group size (15, 16, 17, 31, 32, 33), a many-group request (200) and the 512-split cap
    exercise both combine levels and ragged last groups; fp32 and bf16 outputs."""
    ns_list = [2, 3, 15, 16, 17, 31, 32, 33, 200, 512]
    lens = [16 * n - 5 for n in ns_list] + [0, 7]
    Hkv = 2
    shape, table, q, k, v, ro, rl = _case(lens, Hkv * G, Hkv, seed=20 + G)
    out, lse = _run_gpu(table, q, k, v, chunk_pages=1)
    _check(out, lse, ro, rl)
    ob, lb = _run_gpu(table, q, k, v, chunk_pages=1, out_dtype=l4.L4_DT_BF16)
    assert np.max(np.abs(ob - ro) - np.abs(ro) * 2.0 ** -8) <= TOL
    _check(ob * 0, lb, ro * 0, rl)


def test_workspace_init_and_block_table_layout():
    """A dirty workspace is made usable by l4_decode_workspace_init; a fixed-stride block table
    (indptr[b] = slot_b * max_pages, gaps between requests) is a valid page table (l4.h)."""
    lens = np.array([5, 300, 0, 2048, 17, 999], dtype=np.int64)
    shape, table, q, k, v, ro, rl = _case(lens, 16, 4, seed=31)
    max_pages = 200
    slots = np.array([3, 0, 5, 1, 4, 2])
    bt = np.full(6 * max_pages, -1, dtype=np.int32)
    indptr = np.zeros(7, dtype=np.int32)
    for b in range(6):
        n = table.indptr[b + 1] - table.indptr[b]
        bt[slots[b] * max_pages: slots[b] * max_pages + n] = table.indices[table.indptr[b]:table.indptr[b + 1]]
        indptr[b] = slots[b] * max_pages
    indptr[6] = 6 * max_pages  # not read
    qd, kd, vd = q.cuda(), k.cuda(), v.cuda()
    ip, ix, kl = torch.from_numpy(indptr).cuda(), torch.from_numpy(bt).cuda(), torch.from_numpy(table.kv_len).cuda()
    for flags in (0, l4.L4_DECODE_EARLY_INPUTS):
        params = l4.make_params(6, 16, 4, chunk_pages=3, flags=flags)
        ws = l4.alloc_workspace(params, bt.size)
        ws.fill_(0xFF)  # stale scheduler state and counters
        l4.workspace_init(params, ws)
        out = torch.empty(6, 16, 128, device="cuda")
        lse = torch.empty(6, 16, device="cuda")
        for _ in range(2):
            l4.attention_call(params, qd, kd, vd, ip, ix, kl, bt.size, out, lse, ws)
        torch.cuda.synchronize()
        _check(out.double().cpu().numpy(), lse.double().cpu().numpy(), ro, rl)


def test_validate_page_table():
    """l4_decode_validate flags each kind of page-table corruption and passes a valid table."""
    lens = np.array([5, 300, 0, 2048, 17], dtype=np.int64)
    table = synth.make_page_table(lens, seed=3, spare_pages=10)
    params = l4.make_params(5, 8, 2)
    dev = lambda x: torch.from_numpy(np.ascontiguousarray(x)).cuda()
    assert l4.validate(params, dev(table.kv_len), dev(table.indptr), dev(table.indices), table.num_pages) == (0, -1, 0)
    kl = table.kv_len.copy()
    kl[3] = -1
    assert l4.validate(params, dev(kl), dev(table.indptr), dev(table.indices), table.num_pages) == (1, 3, 1)
    kl = table.kv_len.copy()
    kl[4] = 5000  # runs past the end of the page table
    assert l4.validate(params, dev(kl), dev(table.indptr), dev(table.indices), table.num_pages) == (1, 4, 2)
    ix = table.indices.copy()
    ix[table.indptr[1] + 7] = table.num_pages  # out of the pool
    assert l4.validate(params, dev(table.kv_len), dev(table.indptr), dev(ix), table.num_pages) == (1, 1, 3)
    ix = table.indices.copy()
    ix[table.indptr[3] + 2] = ix[table.indptr[1]]  # request 3 reads request 1's page
    n, first, kind = l4.validate(params, dev(table.kv_len), dev(table.indptr), dev(ix), table.num_pages)
    assert n == 1 and first in (1, 3) and kind == 4
