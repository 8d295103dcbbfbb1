"""paper_2512_19179_b200 — B200-native hot path of L4 (arxiv 2512.19179).

Batched GQA decode attention over paged KV caches with heterogeneous lengths
(length-binned split-KV kernel for sm_100a), the §4.2 stage partition DP and
KV-page migration, behind the C ABI in include/l4.h.  This package is the
thin Python binding; see DESIGN.md.
"""
from .l4 import (  # noqa: F401
    L4_DT_BF16, L4_DT_F32, DecodeParams, KVView, L4Error, NoPagesError, PagePool, alloc_workspace, copy_pages,
    decode_attention, decode_plan, decode_run, enable_peer_access, ipc_close_handle, ipc_get_handle,
    ipc_open_handle, kv_view, lib, make_params, migrate, pack_pages, partition, plan_info, plan_items,
    unpack_pages, version, workspace_size,
)
