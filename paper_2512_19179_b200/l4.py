"""Thin ctypes binding over libl4.so (include/l4.h) — argument marshalling only.

Every computation runs in the native library (CUDA kernels for sm_100a, host
C++ for the partition DP and the page pool).  There is no fallback: if
libl4.so is missing or the device is not a B200, calls raise.
PyTorch supplies device memory, streams and process groups only.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("L4_LIB") or os.path.join(_HERE, "libl4.so")  # L4_LIB: dev-only variant override

L4_OK, L4_ERR_INVALID_ARG, L4_ERR_UNSUPPORTED, L4_ERR_CUDA, L4_ERR_WORKSPACE, L4_ERR_NO_PAGES, L4_ERR_INFEASIBLE = range(7)
L4_DT_F32, L4_DT_BF16 = 0, 1
L4_DECODE_EARLY_INPUTS = 1
L4_DECODE_EARLY_PLAN = 2
_STATUS_NAMES = ["OK", "INVALID_ARG", "UNSUPPORTED", "CUDA", "WORKSPACE", "NO_PAGES", "INFEASIBLE"]

EXPORTED_SYMBOLS = (
    "l4_last_error", "l4_version", "l4_decode_workspace_size", "l4_decode_workspace_init",
    "l4_decode_workspace_regions", "l4_decode_plan", "l4_decode_run",
    "l4_decode_attention", "l4_decode_plan_info", "l4_decode_plan_items", "l4_decode_validate", "l4_partition", "l4_pool_create",
    "l4_pool_alloc", "l4_pool_free", "l4_pool_num_free", "l4_pool_destroy", "l4_migrate", "l4_copy_pages",
    "l4_pack_pages", "l4_unpack_pages", "l4_ipc_get_handle", "l4_ipc_open_handle", "l4_ipc_close_handle",
    "l4_enable_peer_access", "l4_refine_boundary", "l4_qoe_fit",
)


class L4Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        name = _STATUS_NAMES[status] if 0 <= status < len(_STATUS_NAMES) else str(status)
        super().__init__(f"l4 {name}: {msg}")


class NoPagesError(L4Error):
    pass


class DecodeParams(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("num_q_heads", ctypes.c_int32), ("num_kv_heads", ctypes.c_int32),
                ("head_dim", ctypes.c_int32), ("page_size", ctypes.c_int32), ("sm_scale", ctypes.c_float),
                ("out_dtype", ctypes.c_int32), ("chunk_pages", ctypes.c_int32), ("flags", ctypes.c_int32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("num_items", ctypes.c_int32), ("chunk_pages", ctypes.c_int32), ("num_ctas", ctypes.c_int32),
                ("max_splits", ctypes.c_int32), ("tail_requests", ctypes.c_int32),
                ("tail_chunk_pages", ctypes.c_int32)]


class WorkspaceRegions(ctypes.Structure):
    _fields_ = [("state_bytes", ctypes.c_uint64), ("partial_lse_offset", ctypes.c_uint64),
                ("partial_o_offset", ctypes.c_uint64), ("end_offset", ctypes.c_uint64),
                ("items_cap", ctypes.c_int32), ("group_size", ctypes.c_int32)]


class Stage(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_int64), ("hi", ctypes.c_int64), ("instances", ctypes.c_int32)]


class PartitionParams(ctypes.Structure):
    _fields_ = [("num_instances", ctypes.c_int32), ("edges", ctypes.POINTER(ctypes.c_int64)),
                ("num_edges", ctypes.c_int32), ("migrate_bandwidth_Bps", ctypes.c_double),
                ("kv_bytes_per_token", ctypes.c_int64), ("qoe_d", ctypes.c_double * 5),
                ("stage_cost_mode", ctypes.c_int32), ("algorithm", ctypes.c_int32)]


class RefineParams(ctypes.Structure):
    _fields_ = [("qoe_d", ctypes.c_double * 5), ("ema_alpha", ctypes.c_double), ("min_traffic", ctypes.c_int32),
                ("lo", ctypes.c_int64), ("hi", ctypes.c_int64)]


class KVView(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("k_pages", ctypes.c_void_p), ("v_pages", ctypes.c_void_p),
                ("num_pages", ctypes.c_int64), ("num_layers", ctypes.c_int32),
                ("layer_stride_bytes", ctypes.c_int64), ("page_bytes", ctypes.c_int64)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libl4.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not found: build it with `python -m paper_2512_19179_b200.build` "
                          "(no CPU fallback exists)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    P = ctypes.POINTER
    L.l4_last_error.restype = ctypes.c_char_p
    L.l4_version.restype = ctypes.c_char_p
    L.l4_decode_workspace_size.restype = sz
    L.l4_decode_workspace_size.argtypes = [P(DecodeParams), i64]
    L.l4_decode_workspace_init.restype = ctypes.c_int
    L.l4_decode_workspace_init.argtypes = [P(DecodeParams), vp, sz, vp]
    L.l4_decode_workspace_regions.restype = ctypes.c_int
    L.l4_decode_workspace_regions.argtypes = [P(DecodeParams), sz, P(WorkspaceRegions)]
    L.l4_decode_plan.restype = ctypes.c_int
    L.l4_decode_plan.argtypes = [P(DecodeParams), vp, vp, i64, vp, sz, vp]
    L.l4_decode_run.restype = ctypes.c_int
    L.l4_decode_run.argtypes = [P(DecodeParams), vp, vp, vp, i64, vp, vp, vp, vp, sz, vp]
    L.l4_decode_attention.restype = ctypes.c_int
    L.l4_decode_attention.argtypes = [P(DecodeParams), vp, vp, vp, i64, vp, vp, i64, vp, vp, vp, vp, sz, vp]
    L.l4_decode_plan_info.restype = ctypes.c_int
    L.l4_decode_plan_info.argtypes = [vp, P(PlanInfo), vp]
    L.l4_decode_validate.restype = ctypes.c_int
    L.l4_decode_validate.argtypes = [P(DecodeParams), vp, vp, vp, i64, i64, vp, vp, vp]
    L.l4_decode_plan_items.restype = ctypes.c_int
    L.l4_decode_plan_items.argtypes = [vp, vp, i32, vp]
    L.l4_partition.restype = ctypes.c_int
    L.l4_partition.argtypes = [P(PartitionParams), vp, vp, i64, P(Stage), P(i32), P(ctypes.c_double)]
    L.l4_pool_create.restype = ctypes.c_int
    L.l4_pool_create.argtypes = [i64, P(vp)]
    L.l4_pool_alloc.restype = ctypes.c_int
    L.l4_pool_alloc.argtypes = [vp, i64, vp]
    L.l4_pool_free.restype = ctypes.c_int
    L.l4_pool_free.argtypes = [vp, vp, i64]
    L.l4_pool_num_free.restype = i64
    L.l4_pool_num_free.argtypes = [vp]
    L.l4_pool_destroy.restype = None
    L.l4_pool_destroy.argtypes = [vp]
    L.l4_migrate.restype = ctypes.c_int
    L.l4_migrate.argtypes = [P(KVView), vp, i64, P(KVView), vp, vp, vp, vp]
    L.l4_copy_pages.restype = ctypes.c_int
    L.l4_copy_pages.argtypes = [P(KVView), vp, P(KVView), vp, i64, vp]
    L.l4_pack_pages.restype = ctypes.c_int
    L.l4_pack_pages.argtypes = [P(KVView), vp, i64, vp, vp]
    L.l4_unpack_pages.restype = ctypes.c_int
    L.l4_unpack_pages.argtypes = [P(KVView), vp, i64, vp, vp]
    L.l4_ipc_get_handle.restype = ctypes.c_int
    L.l4_ipc_get_handle.argtypes = [vp, vp, P(i64)]
    L.l4_ipc_open_handle.restype = ctypes.c_int
    L.l4_ipc_open_handle.argtypes = [vp, P(vp)]
    L.l4_ipc_close_handle.restype = ctypes.c_int
    L.l4_ipc_close_handle.argtypes = [vp]
    L.l4_qoe_fit.restype = ctypes.c_int
    L.l4_qoe_fit.argtypes = [vp, vp, i64, ctypes.c_uint32, vp, P(ctypes.c_double)]
    L.l4_refine_boundary.restype = ctypes.c_int
    L.l4_refine_boundary.argtypes = [P(RefineParams), vp, vp, i64, i32, vp, vp, vp, ctypes.c_double,
                                     P(ctypes.c_double), P(i64), P(i64)]
    L.l4_enable_peer_access.restype = ctypes.c_int
    L.l4_enable_peer_access.argtypes = [i32]
    _lib = L
    return L


def _check(status: int):
    if status != L4_OK:
        msg = lib().l4_last_error().decode(errors="replace")
        if status == L4_ERR_NO_PAGES:
            raise NoPagesError(status, msg)
        raise L4Error(status, msg)


def version() -> str:
    return lib().l4_version().decode()


# --------------------------------------------------------------------------- helpers

def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_handle(stream) -> Optional[int]:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _need(t, dtype, name, device=True):
    import torch
    if t is None:
        raise ValueError(f"{name} is required")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if device and not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def make_params(batch: int, num_q_heads: int, num_kv_heads: int, head_dim: int = 128, page_size: int = 16,
                sm_scale: float = 0.0, out_dtype: int = L4_DT_F32, chunk_pages: int = 0,
                flags: int = 0) -> DecodeParams:
    return DecodeParams(batch, num_q_heads, num_kv_heads, head_dim, page_size, sm_scale, out_dtype, chunk_pages,
                        flags)


# --------------------------------------------------------------------------- decode attention

def workspace_size(params: DecodeParams, max_total_pages: int) -> int:
    n = lib().l4_decode_workspace_size(ctypes.byref(params), int(max_total_pages))
    if n == 0:
        raise L4Error(L4_ERR_INVALID_ARG, lib().l4_last_error().decode())
    return int(n)


def alloc_workspace(params: DecodeParams, max_total_pages: int, device=None):
    """Device workspace, zero-filled (the scheduler state and split counters must start at 0;
    every call leaves them 0 again)."""
    import torch
    return torch.zeros(workspace_size(params, max_total_pages), dtype=torch.uint8,
                       device=device if device is not None else "cuda")


def workspace_init(params: DecodeParams, workspace, stream=None) -> None:
    """l4_decode_workspace_init: zero the scheduler header and split counters of a workspace."""
    _check(lib().l4_decode_workspace_init(ctypes.byref(params), _ptr(workspace), workspace.numel(),
                                          _stream_handle(stream)))


def workspace_regions(params: DecodeParams, workspace_bytes: int) -> WorkspaceRegions:
    """l4_decode_workspace_regions: byte offsets of the scheduler state and the split partials."""
    r = WorkspaceRegions()
    _check(lib().l4_decode_workspace_regions(ctypes.byref(params), int(workspace_bytes), ctypes.byref(r)))
    return r


def poison_partials(params: DecodeParams, workspace, stream=None) -> None:
    """Debug: fill the split-partial region of a workspace with NaN (0xff bytes), so a combine
    that reads a partial before its split wrote it produces NaN (tests only)."""
    import torch
    r = workspace_regions(params, workspace.numel())
    s = stream if stream is not None else torch.cuda.current_stream()
    with torch.cuda.stream(s):
        workspace[r.partial_lse_offset:r.end_offset].fill_(0xFF)


def decode_plan(params: DecodeParams, kv_len, page_indptr, total_pages: int, workspace, stream=None):
    import torch
    _need(kv_len, torch.int32, "kv_len")
    _need(page_indptr, torch.int32, "page_indptr")
    _check(lib().l4_decode_plan(ctypes.byref(params), _ptr(kv_len), _ptr(page_indptr), int(total_pages),
                                _ptr(workspace), workspace.numel(), _stream_handle(stream)))


def decode_run(params: DecodeParams, q, k_pages, v_pages, page_indices, out, lse, workspace, stream=None):
    import torch
    _need(q, torch.bfloat16, "q")
    _need(k_pages, torch.bfloat16, "k_pages")
    _need(v_pages, torch.bfloat16, "v_pages")
    _need(page_indices, torch.int32, "page_indices")
    _need(out, torch.float32 if params.out_dtype == L4_DT_F32 else torch.bfloat16, "out")
    if lse is not None:
        _need(lse, torch.float32, "lse")
    _check(lib().l4_decode_run(ctypes.byref(params), _ptr(q), _ptr(k_pages), _ptr(v_pages), int(k_pages.shape[0]),
                               _ptr(page_indices), _ptr(out), _ptr(lse), _ptr(workspace), workspace.numel(),
                               _stream_handle(stream)))


def decode_attention(q, k_pages, v_pages, page_indptr, page_indices, kv_len, *, num_kv_heads=None,
                     sm_scale: float = 0.0, out_dtype: int = L4_DT_F32, chunk_pages: int = 0, out=None, lse=None,
                     workspace=None, stream=None, return_lse: bool = True):
    """One decode iteration (plan + run).  q [B,Hq,128] bf16; pools [P,Hkv,16,128] bf16."""
    import torch
    B, Hq, D = q.shape
    Hkv = int(k_pages.shape[1]) if num_kv_heads is None else int(num_kv_heads)
    params = make_params(B, Hq, Hkv, D, int(k_pages.shape[2]), sm_scale, out_dtype, chunk_pages)
    total_pages = int(page_indices.numel())
    if workspace is None:
        workspace = alloc_workspace(params, total_pages, q.device)
    if out is None:
        out = torch.empty(B, Hq, D, dtype=torch.float32 if out_dtype == L4_DT_F32 else torch.bfloat16,
                          device=q.device)
    if lse is None and return_lse:
        lse = torch.empty(B, Hq, dtype=torch.float32, device=q.device)
    attention_call(params, q, k_pages, v_pages, page_indptr, page_indices, kv_len, total_pages, out, lse,
                   workspace, stream)
    return out, lse


def attention_call(params: DecodeParams, q, k_pages, v_pages, page_indptr, page_indices, kv_len, total_pages: int,
                   out, lse, workspace, stream=None):
    """l4_decode_attention: plan + split-KV + combine in one launch (B <= 1024)."""
    import torch
    _need(q, torch.bfloat16, "q")
    _need(k_pages, torch.bfloat16, "k_pages")
    _need(v_pages, torch.bfloat16, "v_pages")
    _need(page_indptr, torch.int32, "page_indptr")
    _need(page_indices, torch.int32, "page_indices")
    _need(kv_len, torch.int32, "kv_len")
    _need(out, torch.float32 if params.out_dtype == L4_DT_F32 else torch.bfloat16, "out")
    if lse is not None:
        _need(lse, torch.float32, "lse")
    _check(lib().l4_decode_attention(ctypes.byref(params), _ptr(q), _ptr(k_pages), _ptr(v_pages),
                                     int(k_pages.shape[0]), _ptr(page_indptr), _ptr(page_indices), int(total_pages),
                                     _ptr(kv_len), _ptr(out), _ptr(lse), _ptr(workspace), workspace.numel(),
                                     _stream_handle(stream)))


def validate(params: DecodeParams, kv_len, page_indptr, page_indices, num_pages: int, stream=None):
    """l4_decode_validate (debug): returns (violations, first offending request, kind) with kind
    1 length < 0, 2 indptr range, 3 page id range, 4 page read by two requests / twice."""
    import torch
    _need(kv_len, torch.int32, "kv_len")
    _need(page_indptr, torch.int32, "page_indptr")
    _need(page_indices, torch.int32, "page_indices")
    scratch = torch.empty(max(int(num_pages), 1) + 2, dtype=torch.int32, device=kv_len.device)
    rep = (ctypes.c_int32 * 3)()
    _check(lib().l4_decode_validate(ctypes.byref(params), _ptr(kv_len), _ptr(page_indptr), _ptr(page_indices),
                                    int(page_indices.numel()), int(num_pages), _ptr(scratch), rep,
                                    _stream_handle(stream)))
    return int(rep[0]), int(rep[1]), int(rep[2])


def plan_info(workspace, stream=None) -> PlanInfo:
    info = PlanInfo()
    _check(lib().l4_decode_plan_info(_ptr(workspace), ctypes.byref(info), _stream_handle(stream)))
    return info


def plan_items(workspace, stream=None) -> np.ndarray:
    info = plan_info(workspace, stream)
    buf = np.zeros((max(info.num_items, 0), 8), dtype=np.int32)
    if info.num_items > 0:
        _check(lib().l4_decode_plan_items(_ptr(workspace), buf.ctypes.data, info.num_items, _stream_handle(stream)))
    return buf


# --------------------------------------------------------------------------- partition (host)

PART_EXACT, PART_CHAIN, PART_TWO_PHASE = 0, 1, 2


def partition(input_len: Sequence[int], output_len: Sequence[int], num_instances: int, qoe_d,
              bandwidth_Bps: float, kv_bytes_per_token: int, edges=None, mode: int = 0, chain: bool = False,
              algorithm: int = PART_EXACT):
    """l4_partition: returns ([(lo, hi, instances)], objective).  algorithm: 0 exact DP,
    1 chain DP (also selected by chain=True), 2 two-phase heuristic."""
    I = np.ascontiguousarray(np.asarray(input_len, dtype=np.int64))
    O = np.ascontiguousarray(np.asarray(output_len, dtype=np.int64))
    if I.shape != O.shape:
        raise ValueError("input_len and output_len differ in length")
    p = PartitionParams()
    p.num_instances = int(num_instances)
    edges_arr = None
    if edges is not None:
        edges_arr = np.ascontiguousarray(np.asarray(edges, dtype=np.int64))
        p.edges = edges_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
        p.num_edges = int(edges_arr.size)
    p.migrate_bandwidth_Bps = float(bandwidth_Bps)
    p.kv_bytes_per_token = int(kv_bytes_per_token)
    for k in range(5):
        p.qoe_d[k] = float(qoe_d[k])
    p.stage_cost_mode = int(mode)
    p.algorithm = PART_CHAIN if chain else int(algorithm)
    cap = max(int(num_instances), 1)
    stages = (Stage * cap)()
    ns = ctypes.c_int32(0)
    obj = ctypes.c_double(0.0)
    _check(lib().l4_partition(ctypes.byref(p), I.ctypes.data if I.size else None, O.ctypes.data if O.size else None,
                              int(I.size), stages, ctypes.byref(ns), ctypes.byref(obj)))
    return [(int(stages[k].lo), int(stages[k].hi), int(stages[k].instances)) for k in range(ns.value)], obj.value


def qoe_fit(F, Q, mask=(1, 1, 1, 1, 1)):
    """l4_qoe_fit: returns (D[5], rms residual)."""
    Fa = np.ascontiguousarray(np.asarray(F, dtype=np.float64).reshape(-1, 5))
    Qa = np.ascontiguousarray(np.asarray(Q, dtype=np.float64).reshape(-1))
    bits = sum(1 << k for k in range(5) if mask[k])
    D = np.zeros(5)
    rms = ctypes.c_double(0.0)
    _check(lib().l4_qoe_fit(Fa.ctypes.data, Qa.ctypes.data, int(Qa.size), bits, D.ctypes.data, ctypes.byref(rms)))
    return D, rms.value


def refine_boundary(boundary: float, local, successor_sets, qoe_d, alpha: float = 0.3, min_traffic: int = 5,
                    lo: int = 0, hi: int = 1 << 62):
    """l4_refine_boundary: local = [(I, L)], successor_sets = [[(I, L)], ...].
    Returns (new boundary, raw split length or None, split index or None)."""
    loc = np.asarray(list(local), dtype=np.int64).reshape(-1, 2)
    sets = [np.asarray(list(s), dtype=np.int64).reshape(-1, 2) for s in successor_sets]
    indptr = np.zeros(len(sets) + 1, dtype=np.int64)
    for k, s in enumerate(sets):
        indptr[k + 1] = indptr[k] + len(s)
    allsucc = np.concatenate(sets) if sets and indptr[-1] > 0 else np.zeros((0, 2), dtype=np.int64)
    lI, lL = np.ascontiguousarray(loc[:, 0]), np.ascontiguousarray(loc[:, 1])
    sI, sL = np.ascontiguousarray(allsucc[:, 0]), np.ascontiguousarray(allsucc[:, 1])
    p = RefineParams()
    for k in range(5):
        p.qoe_d[k] = float(qoe_d[k])
    p.ema_alpha, p.min_traffic, p.lo, p.hi = float(alpha), int(min_traffic), int(lo), int(hi)
    out_b, raw, split = ctypes.c_double(0), ctypes.c_int64(0), ctypes.c_int64(0)
    ptr = lambda a: a.ctypes.data if a.size else None
    _check(lib().l4_refine_boundary(ctypes.byref(p), ptr(lI), ptr(lL), int(lI.size), len(sets),
                                    indptr.ctypes.data if sets else None, ptr(sI), ptr(sL), float(boundary),
                                    ctypes.byref(out_b), ctypes.byref(raw), ctypes.byref(split)))
    return out_b.value, (None if raw.value < 0 else int(raw.value)), (None if split.value < 0 else int(split.value))


# --------------------------------------------------------------------------- page pool + migration

class PagePool:
    """Host-side lowest-free-first page allocator (l4_pool_*)."""

    def __init__(self, num_pages: int):
        h = ctypes.c_void_p()
        _check(lib().l4_pool_create(int(num_pages), ctypes.byref(h)))
        self._h = h
        self.num_pages = int(num_pages)

    @property
    def handle(self):
        return self._h

    def alloc(self, n: int) -> np.ndarray:
        out = np.zeros(int(n), dtype=np.int32)
        _check(lib().l4_pool_alloc(self._h, int(n), out.ctypes.data if n else None))
        return out

    def free(self, pages) -> None:
        arr = np.ascontiguousarray(np.asarray(pages, dtype=np.int32))
        _check(lib().l4_pool_free(self._h, arr.ctypes.data if arr.size else None, int(arr.size)))

    def num_free(self) -> int:
        return int(lib().l4_pool_num_free(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.l4_pool_destroy(h)
            self._h = None


def kv_view(k_pages, v_pages, device: Optional[int] = None, num_layers: int = 1, num_pages: Optional[int] = None,
            layer_stride_bytes: Optional[int] = None, page_bytes: Optional[int] = None,
            k_ptr: Optional[int] = None, v_ptr: Optional[int] = None) -> KVView:
    """KV view over pools shaped [layers, num_pages, ...] or [num_pages, ...] (torch tensors), or raw pointers."""
    if k_pages is not None:
        if num_layers > 1:
            L, P = int(k_pages.shape[0]), int(k_pages.shape[1])
            assert L == num_layers
            pb = int(k_pages[0, 0].numel() * k_pages.element_size())
            stride = int(k_pages.stride(0) * k_pages.element_size())
        else:
            P = int(k_pages.shape[0])
            pb = int(k_pages[0].numel() * k_pages.element_size())
            stride = P * pb
        k_ptr, v_ptr = k_pages.data_ptr(), v_pages.data_ptr()
        num_pages = P if num_pages is None else num_pages
        page_bytes = pb if page_bytes is None else page_bytes
        layer_stride_bytes = stride if layer_stride_bytes is None else layer_stride_bytes
        device = k_pages.device.index if device is None else device
    return KVView(int(device or 0), k_ptr, v_ptr, int(num_pages), int(num_layers), int(layer_stride_bytes),
                  int(page_bytes))


def migrate(src: KVView, src_pages, dst: KVView, dst_pool: PagePool, stream=None, done_event=None) -> np.ndarray:
    sp = np.ascontiguousarray(np.asarray(src_pages, dtype=np.int32))
    out = np.zeros(sp.size, dtype=np.int32)
    ev = None if done_event is None else done_event.cuda_event
    _check(lib().l4_migrate(ctypes.byref(src), sp.ctypes.data if sp.size else None, int(sp.size), ctypes.byref(dst),
                            dst_pool.handle, out.ctypes.data if sp.size else None, _stream_handle(stream), ev))
    return out


def copy_pages(src: KVView, src_pages, dst: KVView, dst_pages, stream=None) -> None:
    sp = np.ascontiguousarray(np.asarray(src_pages, dtype=np.int32))
    dp = np.ascontiguousarray(np.asarray(dst_pages, dtype=np.int32))
    assert sp.size == dp.size
    _check(lib().l4_copy_pages(ctypes.byref(src), sp.ctypes.data if sp.size else None, ctypes.byref(dst),
                               dp.ctypes.data if dp.size else None, int(sp.size), _stream_handle(stream)))


def pack_pages(src: KVView, pages, staging, stream=None) -> None:
    p = np.ascontiguousarray(np.asarray(pages, dtype=np.int32))
    _check(lib().l4_pack_pages(ctypes.byref(src), p.ctypes.data if p.size else None, int(p.size), _ptr(staging),
                               _stream_handle(stream)))


def unpack_pages(dst: KVView, pages, staging, stream=None) -> None:
    p = np.ascontiguousarray(np.asarray(pages, dtype=np.int32))
    _check(lib().l4_unpack_pages(ctypes.byref(dst), p.ctypes.data if p.size else None, int(p.size), _ptr(staging),
                                 _stream_handle(stream)))


def ipc_get_handle(ptr: int):
    """(64-byte handle of the allocation containing ptr, ptr's offset in it)."""
    buf = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _check(lib().l4_ipc_get_handle(ptr, buf, ctypes.byref(off)))
    return buf.raw, int(off.value)


def ipc_open_handle(handle: bytes) -> int:
    assert len(handle) == 64
    out = ctypes.c_void_p()
    _check(lib().l4_ipc_open_handle(handle, ctypes.byref(out)))
    return int(out.value)


def ipc_close_handle(ptr: int) -> None:
    _check(lib().l4_ipc_close_handle(ptr))


def enable_peer_access(peer_device: int) -> None:
    _check(lib().l4_enable_peer_access(int(peer_device)))
