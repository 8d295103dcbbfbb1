/*
 * l4.h — C ABI of the B200-native L4 hot path (arxiv 2512.19179, "L4: Low-Latency
 * and Load-Balanced LLM Serving via Length-Aware Scheduling").
 *
 * Citations: "P:n" = /root/reference/PAPER.md line n, "S:n" = SPEC.md line n,
 * "Zk" = reading k of DESIGN.md §Readings.
 *
 * Conventions (apply to every call unless stated otherwise)
 *  - Every call returns l4_status and never throws or aborts.  On error a
 *    description is available from l4_last_error() on the same thread.
 *  - Errors leave no side effects: outputs are written only on L4_OK.
 *  - Ownership: the caller owns every buffer.  The library never allocates
 *    device memory on the hot path (workspaces are passed in) and keeps no
 *    pointer after return.  The only library-owned objects are l4_page_pool
 *    handles.
 *  - Device work is enqueued on the caller's stream ("stream" is a
 *    cudaStream_t passed as void*; NULL = legacy default stream) and is
 *    asynchronous; kernel faults surface at the caller's next synchronisation.
 *  - Host-checkable arguments are validated synchronously.
 *  - There is no CPU fallback and no multi-backend dispatch: the device path
 *    is sm_100a only (B200).  On a host without such a device, device calls
 *    return L4_ERR_CUDA.
 */
#ifndef L4_H
#define L4_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  L4_OK = 0,
  L4_ERR_INVALID_ARG = 1,  /* a host-checkable argument is out of range / NULL */
  L4_ERR_UNSUPPORTED = 2,  /* valid but not implemented (e.g. head_dim != 128) */
  L4_ERR_CUDA = 3,         /* a CUDA runtime/driver call failed (no device, launch error) */
  L4_ERR_WORKSPACE = 4,    /* workspace NULL or smaller than l4_decode_workspace_size() */
  L4_ERR_NO_PAGES = 5,     /* destination pool has no idle pages; nothing changed */
  L4_ERR_INFEASIBLE = 6    /* partition edges do not cover every request (Z10) */
} l4_status;

/* Thread-local description of the last error on this thread; valid until the
 * next l4_* call on the same thread.  Never NULL. */
const char* l4_last_error(void);
/* Library version string, e.g. "l4-b200 0.1.0 sm_100a". */
const char* l4_version(void);

/* ========================================================================
 * 1. Decode attention over a paged KV cache
 *
 * One decode iteration for a batch of B requests: for request b with kv_len
 * L_b and q-head h (kv head g = h / G, G = Hq/Hkv, Z18):
 *   s_t = scale * <q[b,h,:], K_t>,  t in [0, L_b)           (Z20)
 *   out[b,h,:] = sum_t softmax(s)_t V_t,  lse[b,h] = ln sum_t exp(s_t)  (Z22)
 * where token t lives at page indices[indptr[b] + t/16], slot t%16 (Z19).
 * L_b = 0 gives out = 0 and lse = -inf (Z21).
 *
 * Layout (Z19): K and V pools are separate bf16 arrays [num_pages, Hkv, 16, 128]
 * ("HND": each (page, kv head) slice is 16 x 128 bf16 = 4 KB contiguous).
 * q is bf16 [B, Hq, 128]; out is [B, Hq, 128] f32 or bf16; lse f32 [B, Hq].
 * Page table: int32 indptr [B+1], indices, kv_len [B].  Request b's page ids are
 * indices[indptr[b] .. indptr[b] + ceil(L_b/16)); only those entries are read, so a
 * compact CSR (indptr non-decreasing) and a fixed-stride block table
 * (indptr[b] = slot_b * max_pages) are both valid.
 *
 * Method (the paper's problem, B200 design in DESIGN.md §Kernels): a device
 * planner builds LENGTH-BINNED work lists (each request's pages are split
 * into near-equal chunks, items are ordered by descending chunk size so long
 * and short sequences do not stall each other); a persistent
 * split-KV kernel streams (page, kv head) slices with TMA into a shared-memory
 * ring, computes QK^T and PV on tensor cores with an online softmax, and the
 * last split of each (request, kv head) performs the log-sum-exp combine
 * (FlashDecoding aggregation).
 * ======================================================================== */

enum { L4_DT_F32 = 0, L4_DT_BF16 = 1 };

typedef struct {
  int32_t batch;          /* B >= 0, <= 8192 */
  int32_t num_q_heads;    /* Hq >= 1 */
  int32_t num_kv_heads;   /* Hkv >= 1, Hq % Hkv == 0, G = Hq/Hkv in {1,2,4,8} */
  int32_t head_dim;       /* must be 128 (else L4_ERR_UNSUPPORTED) */
  int32_t page_size;      /* must be 16  (else L4_ERR_UNSUPPORTED) */
  float   sm_scale;       /* <= 0 -> 1/sqrt(head_dim) (Z17) */
  int32_t out_dtype;      /* L4_DT_F32 (parity) or L4_DT_BF16 */
  int32_t chunk_pages;    /* 0 = automatic length-binned split; > 0 forces the split
                             chunk C (pages per work item); < 0 = never split.  Requests
                             of <= 2C pages are never split (no combine needed). */
  int32_t flags;          /* 0, L4_DECODE_EARLY_PLAN or L4_DECODE_EARLY_INPUTS (below) */
} l4_decode_params;

/* l4_decode_attention (single-launch path) may start reading its INPUTS (q, the KV pools,
 * kv_len, page_indptr, page_indices) while the previous kernel on the stream is still
 * running (programmatic dependent launch), so in a loop of calls the next call's planning
 * and first page loads overlap the previous call's tail.  Outputs and the workspace are
 * still touched only after the previous kernel has completed.  Set it only when the kernel
 * launched immediately before on the same stream cannot be writing those inputs (another
 * l4 call, or any kernel that does not itself trigger programmatic launch early). */
enum { L4_DECODE_EARLY_INPUTS = 1 };
/* Weaker form for a decode step's layer loop, where the kernel before attention writes q and the
 * step's new K/V token but never the page table: only the planner's inputs (kv_len, page_indptr)
 * are read before the previous kernel completes; q, the KV pools, page_indices, the workspace and
 * the outputs are touched after it.  Set it only when the kernel launched immediately before on
 * the same stream cannot be writing kv_len / page_indptr.  L4_DECODE_EARLY_INPUTS implies it. */
enum { L4_DECODE_EARLY_PLAN = 2 };
/* Without either flag nothing is read before the previous kernel completes; the kernel only issues
 * L2 prefetch hints (cp.async.bulk.prefetch.L2) for page_indices, q, kv_len and page_indptr as its
 * CTAs start, which cannot return stale data (L2 is the point of coherence). */

/* Bytes of device workspace needed for any batch whose page table has at most
 * max_total_pages entries (indptr[B] <= max_total_pages).  Returns 0 if the
 * params are invalid (see l4_last_error()).  Must be queried with the target
 * device current (the bound depends on its SM count).
 * A workspace is caller-owned device memory.  It must be zero-filled once before its
 * first use (l4_decode_workspace_init, or any zero fill); every completed call leaves
 * its scheduler state and split counters zero again, so it can then be reused by any
 * number of calls with the same num_kv_heads and any batch <= 8192. */
size_t l4_decode_workspace_size(const l4_decode_params* p, int64_t max_total_pages);

/* Zero the workspace's scheduler header and split counters (cudaMemsetAsync on `stream`). */
l4_status l4_decode_workspace_init(const l4_decode_params* p, void* workspace, size_t workspace_bytes,
                                   void* stream);

/* Byte regions of a workspace of `workspace_bytes` (host-only, no device access; diagnostics
 * and tests).  [0, state_bytes) holds the scheduler header and the split counters (must be
 * zero between calls); [partial_lse_offset, +items_cap*G*4) the base-2 LSE of the split
 * partials and [partial_o_offset, +items_cap*G*128*4) their normalised outputs (fp32), both
 * indexed by work item.  Nothing in the partial regions survives a call as state: a test may
 * fill them with NaN before every call so that a combine reading a partial before it was
 * written shows up as NaN.  Errors: INVALID_ARG (params), WORKSPACE (too small). */
typedef struct {
  uint64_t state_bytes;
  uint64_t partial_lse_offset;
  uint64_t partial_o_offset;
  uint64_t end_offset;          /* end of the partial region (<= workspace_bytes) */
  int32_t  items_cap;           /* work-item / partial-slot capacity */
  int32_t  group_size;          /* G = Hq / Hkv */
} l4_workspace_regions;
l4_status l4_decode_workspace_regions(const l4_decode_params* p, size_t workspace_bytes,
                                      l4_workspace_regions* out);

/* a1: build the length-binned work list for this step from device kv_len [B]
 * and page_indptr [B+1] into `workspace` (one device kernel, graph-capturable,
 * no host synchronisation).  The plan stays valid for any number of
 * l4_decode_run calls with the same page table (e.g. every layer of a step). */
l4_status l4_decode_plan(const l4_decode_params* p, const int32_t* kv_len, const int32_t* page_indptr,
                         int64_t total_pages, void* workspace, size_t workspace_bytes, void* stream);

/* a2+a3: run the split-KV kernel (with its fused LSE combine) for the plan in
 * `workspace`.  k_pages/v_pages: device bf16 pools of num_pages pages;
 * page_indices: device int32 [total_pages]; out: device [B,Hq,128] of
 * p->out_dtype; lse: device f32 [B,Hq] or NULL.  Page ids must lie in
 * [0, num_pages) (an id outside reads zeros, never out of bounds). */
l4_status l4_decode_run(const l4_decode_params* p, const void* q, const void* k_pages, const void* v_pages,
                        int64_t num_pages, const int32_t* page_indices, void* out, float* lse,
                        void* workspace, size_t workspace_bytes, void* stream);

/* One decode iteration in ONE kernel launch (a1 + a2 + a3): for B <= 1024 every CTA of the
 * persistent split-KV kernel builds the same length-binned plan in its own shared memory
 * from kv_len / page_indptr (no planner launch, no global work list, no host sync); larger
 * batches run l4_decode_plan then l4_decode_run.  Identical results to plan + run (same
 * work list, same reduction order).  Does not leave a reusable plan in the workspace:
 * call l4_decode_plan before l4_decode_run. */
l4_status l4_decode_attention(const l4_decode_params* p, const void* q, const void* k_pages,
                              const void* v_pages, int64_t num_pages, const int32_t* page_indptr,
                              const int32_t* page_indices, int64_t total_pages, const int32_t* kv_len,
                              void* out, float* lse, void* workspace, size_t workspace_bytes, void* stream);

/* Plan statistics (for tests/benchmarks): copies the plan header from the
 * workspace to the host, synchronising `stream`.  NOT for the hot path. */
typedef struct {
  int32_t num_items;      /* work items (request, kv head, page chunk) */
  int32_t chunk_pages;    /* chunk chosen by the planner */
  int32_t num_ctas;       /* persistent grid of l4_decode_run */
  int32_t max_splits;     /* largest split count of any request (before the guided tail) */
  int32_t tail_requests;  /* requests of the guided tail (split finer, processed last) */
  int32_t tail_chunk_pages; /* chunk of the guided tail (0 if none) */
} l4_plan_info;
l4_status l4_decode_plan_info(const void* workspace, l4_plan_info* info_out, void* stream);

/* Copy the planner's work list (int32 x 8 per item: b, kv_head, abs page begin,
 * abs page end, valid tokens in last page, part base, n splits, split index)
 * to host memory `items_out` (capacity max_items).  Synchronises `stream`.
 * Test/diagnostic use only. */
l4_status l4_decode_plan_items(const void* workspace, int32_t* items_out, int32_t max_items, void* stream);

/* Debug check of a page table before decode (the hot path trusts it): on the device, for every
 * request b: kv_len[b] >= 0; indptr[b] >= 0 and indptr[b] + ceil(kv_len[b]/16) <= total_pages;
 * every page id the request reads lies in [0, num_pages); and no page id is read by two
 * requests or twice by one (a page belongs to one sequence).  Writes to host `report`:
 * [0] number of violations, [1] first offending request (or -1), [2] its violation kind
 * (1 length, 2 indptr range, 3 page id range, 4 page shared).  Synchronises `stream`.  The
 * check uses `scratch` (device, >= num_pages + 2 int32, overwritten): a page-owner table and
 * the device-side report. */
l4_status l4_decode_validate(const l4_decode_params* p, const int32_t* kv_len, const int32_t* page_indptr,
                             const int32_t* page_indices, int64_t total_pages, int64_t num_pages,
                             int32_t* scratch, int32_t* report, void* stream);

/* ========================================================================
 * 2. Length-aware stage partition (§4.2) — host code
 *
 * The DP  f_{s,e,l} = min_{e',l'} f_{s-1,e',l'} + (e-e') Q^{n_{l',l}/(e-e')} + c_{l'}
 * over exponential bucket edges with the batch QoE of
 * Eq. (1) and cut cost c_{l'} = straddling tokens * bytes / bandwidth
 * (P:341).  Requests are members of the range of their final length I+O (Z4),
 * sorted by (I+O, I, index) (Z6).  Ties: smaller e', then smaller l' (Z11),
 * then fewer stages (Z12).  Bit-exact with oracle/partition.py (Z14) for every algorithm.
 * ======================================================================== */

typedef struct {
  int64_t lo;             /* inclusive length bound (tokens) */
  int64_t hi;             /* exclusive length bound */
  int32_t instances;      /* >= 1 */
} l4_stage;

typedef struct {
  int32_t num_instances;        /* E >= 1 */
  const int64_t* edges;         /* NULL -> 0,1,2,4,...,2^K with 2^K > max(I+O) (Z10);
                                   else strictly increasing, edges[0] = 0, last > max(I+O) */
  int32_t num_edges;            /* entries in edges (>= 2) when edges != NULL */
  double  migrate_bandwidth_Bps;/* > 0, bytes per second */
  int64_t kv_bytes_per_token;   /* >= 0, e.g. 2*Hkv*D*2*layers */
  double  qoe_d[5];             /* D_0..D_4 of Eq. (1) */
  int32_t stage_cost_mode;      /* 0 = paper-literal footnote (Z5/Z7); 1 = exact strided split */
  int32_t algorithm;            /* 0 = exact DP (default); 1 = chain DP, one instance per stage;
                                   2 = two-phase heuristic: chain DP + greedy adjacent merges with the
                                   largest positive gain, max-heap (readings Z31-Z33) */
} l4_partition_params;

/* input_len/output_len: host int64 [n], each >= 1.  stages_out: capacity >= E.
 * Writes the stages in ascending length order, their count and the objective
 * (min over s of f_{s,E,top}).  Errors: INVALID_ARG, INFEASIBLE (edges do not
 * cover all final lengths). */
l4_status l4_partition(const l4_partition_params* p, const int64_t* input_len, const int64_t* output_len,
                       int64_t n, l4_stage* stages_out, int32_t* num_stages_out, double* objective_out);

/* §4.1 QoE model fit: least-squares D_0..D_4 with Q^(j) ~ sum_k D_k F_k^(j).
 * F: host row-major [n, 5] features (1, n, sum I, sum I^2, sum L) per sample; Q: [n] observed
 * per-request latency.  column_mask bit k selects F_k (reading Z38: decode-only profiles use
 * 0b10011 = {1, n, sum L}); unselected D_k = 0.  Householder QR on scaled columns.
 * Errors: n < selected columns -> INVALID_ARG; rank deficient -> INFEASIBLE.
 * rms_out (nullable): root-mean-square residual. */
l4_status l4_qoe_fit(const double* F, const double* Q, int64_t n, uint32_t column_mask, double* D_out,
                     double* rms_out);

/* §4.3 adaptive range refinement (readings Z34-Z37): refine the boundary
 * between a stage [lo, boundary) and its successor [boundary, hi).  The successors'
 * (I, L) sets (CSR: succ_indptr [n_succ+1], succ_I / succ_L) are averaged with the
 * §4.2 set division, merged with the local (I, L) list and sorted by (L, I) into R;
 * b = argmin_{0<=i<N} Q^{R[:i]} + Q^{R[i:]} (Eq. (1), smallest i on ties); the boundary
 * moves by an exponential moving average towards R[b].L and is clamped to
 * [lo+1, hi-1].  With fewer than min_traffic merged requests it is left unchanged
 * (raw_out = split_out = -1).  Bit-exact with oracle/refine.py. */
typedef struct {
  double  qoe_d[5];       /* D_0..D_4 of Eq. (1) */
  double  ema_alpha;      /* in [0, 1] */
  int32_t min_traffic;    /* freeze below this many requests (paper: five) */
  int64_t lo, hi;         /* outer bounds: the stage's lo and the successor stage's hi */
} l4_refine_params;
l4_status l4_refine_boundary(const l4_refine_params* p, const int64_t* local_I, const int64_t* local_L,
                             int64_t n_local, int32_t n_succ, const int64_t* succ_indptr, const int64_t* succ_I,
                             const int64_t* succ_L, double boundary_in, double* boundary_out, int64_t* raw_out,
                             int64_t* split_out);

/* ========================================================================
 * 3. KV page pool and migration
 * ======================================================================== */

/* Host-side page allocator over ids 0..num_pages-1: deterministic
 * lowest-free-first (Z27), all-or-nothing. */
typedef struct l4_page_pool l4_page_pool;
l4_status l4_pool_create(int64_t num_pages, l4_page_pool** out);
/* n lowest free ids, ascending, into pages_out; L4_ERR_NO_PAGES leaves the pool unchanged (Z28). */
l4_status l4_pool_alloc(l4_page_pool* pool, int64_t n, int32_t* pages_out);
/* Free n ids; an id out of range, already free, or repeated -> INVALID_ARG, pool unchanged. */
l4_status l4_pool_free(l4_page_pool* pool, const int32_t* pages, int64_t n);
int64_t   l4_pool_num_free(const l4_page_pool* pool);
void      l4_pool_destroy(l4_page_pool* pool);

/* A device KV cache: for layer l and page p, the K slice starts at
 * k_pages + l*layer_stride_bytes + p*page_bytes (V likewise).  page_bytes =
 * Hkv*16*128*2 for the decode layout; must be a multiple of 16.  Pointers may
 * be local or peer / IPC-mapped addresses of another GPU. */
typedef struct {
  int32_t device;             /* CUDA ordinal that owns the memory (informational) */
  void*   k_pages;
  void*   v_pages;
  int64_t num_pages;
  int32_t num_layers;         /* >= 1 */
  int64_t layer_stride_bytes; /* >= num_pages*page_bytes when num_layers > 1 */
  int64_t page_bytes;
} l4_kv_view;

/* a5: one request's KV pages src -> dst (one-sided push).  Allocates n_pages
 * destination pages lowest-free-first from dst_pool (all-or-nothing; no idle
 * cache -> L4_ERR_NO_PAGES and nothing is copied), writes their ids to
 * dst_pages_out (host), then enqueues ONE kernel on `stream` (issued on the
 * current device, which must be able to address both views) that copies every
 * page's K and V slices of every layer straight into the destination slots
 * (no staging buffer).  If done_event (cudaEvent_t) is non-NULL it is
 * recorded after the copy.  The caller frees the source pages only after the
 * copy completed (exactly-once ownership).  src_pages: host int32 [n].
 * Errors after the allocation: a failed launch returns L4_ERR_CUDA with the destination pages
 * back in the pool once the copies already enqueued have drained (if that synchronisation also
 * fails they stay allocated and their ids are in dst_pages_out); a failed cudaEventRecord returns
 * L4_ERR_CUDA with the copy enqueued and the allocated ids in dst_pages_out. */
l4_status l4_migrate(const l4_kv_view* src, const int32_t* src_pages, int64_t n_pages, const l4_kv_view* dst,
                     l4_page_pool* dst_pool, int32_t* dst_pages_out, void* stream, void* done_event);

/* Same copy with explicit host page lists (no allocation). */
l4_status l4_copy_pages(const l4_kv_view* src, const int32_t* src_pages, const l4_kv_view* dst,
                        const int32_t* dst_pages, int64_t n_pages, void* stream);

/* Two-sided building blocks (send/recv by the caller, e.g. NCCL):
 * staging is device memory of n*num_layers*2*page_bytes bytes, ordered
 * [page i][layer][K,V][page_bytes]. */
l4_status l4_pack_pages(const l4_kv_view* src, const int32_t* pages, int64_t n, void* staging, void* stream);
l4_status l4_unpack_pages(const l4_kv_view* dst, const int32_t* pages, int64_t n, const void* staging,
                          void* stream);

/* CUDA IPC helpers for the cross-process one-sided path (one process per GPU): a process
 * exports its KV pools, a peer maps them and l4_copy_pages / l4_migrate write straight into
 * them.  The handle names the whole device allocation containing dev_ptr; offset_out
 * (nullable) receives dev_ptr - allocation base, to add to the pointer l4_ipc_open_handle
 * returns (pools from a caching allocator are sub-allocations). */
enum { L4_IPC_HANDLE_BYTES = 64 };
l4_status l4_ipc_get_handle(const void* dev_ptr, void* handle_out /* 64 bytes */, int64_t* offset_out);
l4_status l4_ipc_open_handle(const void* handle /* 64 bytes */, void** dev_ptr_out);
l4_status l4_ipc_close_handle(void* dev_ptr);
/* Enable peer access from the current device to peer_device (idempotent). */
l4_status l4_enable_peer_access(int32_t peer_device);

#ifdef __cplusplus
}
#endif

#endif /* L4_H */
