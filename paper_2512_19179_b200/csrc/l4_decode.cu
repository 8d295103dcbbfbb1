// l4_decode: length-binned split-KV GQA decode attention over a paged KV cache,
// for B200 (sm_100a).  Entry points: l4_decode_workspace_size / _plan / _run /
// _attention in include/l4.h.
//
// What is computed (definition in oracle/attention.py): for
// every request b and q-head h, softmax(scale * q K^T) V over the L_b cached
// tokens of kv head h/G, plus the natural-log LSE.
//
// How (B200 design):
//  a1  plan_core: pages -> chunk size C -> near-equal splits of the requests
//      longer than 2C -> work items binned by split length, longest bin first
//      (LPT order), so the longest request's splits start first and short
//      requests fill the tail (the paper's inter-SM imbalance and partitioning
//      inefficiency).  Run by EVERY CTA of the single-launch path
//      (l4_decode_attention: the plan stays in shared memory, no planner launch)
//      or by plan_kernel (l4_decode_plan: a materialised work list reused by
//      l4_decode_run, e.g. for every layer of a step).  Unsplit single-bin
//      batches skip the sort; large all-split batches pick the chunk whose last
//      round of items is ~85% full (chunk_search).
//  a2  decode_kernel (persistent, 1 producer + 4 consumer warps per CTA,
//      2 CTAs per SM): items are handed out dynamically (first one static,
//      then one atomic ticket per unit), so CTAs that finish early
//      take the next-largest item.  The producer warp streams each (page, kv
//      head) K and V slice (4 KB each, HND layout) with one TMA each
//      (cp.async.bulk.tensor, 128B swizzle, L2 evict-first) into an 8-stage
//      shared-memory ring tracked by mbarriers; consumer warps compute
//      S^T = K Q^T and O^T += V^T P^T with mma.sync m16n8k16 (tokens / head_dim
//      on M, the G <= 8 query heads on N, so GQA group 8 has no padding), an
//      online softmax with warp-shuffle max reductions in the exp2 domain, and
//      P split into bf16 hi + lo (Z23); a stage goes back to the producer as
//      soon as its K and V fragments are in registers.  With
//      L4_DECODE_EARLY_INPUTS the next call plans and streams its first item
//      while this one finishes (PDL); every call issues L2 prefetch hints for
//      its first inputs at entry.  Quad units: when the short unsplit items at
//      the end of the LPT order are numerous enough (clamp(pages / 10, 1, 4)
//      units of four per CTA), they are handed out four at a time, one whole
//      item per consumer warp (pages of the four items interleaved in the ring;
//      the next unit's ticket and page ids fetched while this one's pages go
//      out), with no cross-warp merge or CTA barrier per item: short-request
//      batches stop paying a merge per few pages.
//  a3  LSE combine: the 4 warps of a CTA merge their (m, l, O) in shared
//      memory; a split item writes (O/l, lse) to the workspace; the last split
//      of each group of 16 combines the group, the last group combines the
//      groups (FlashDecoding aggregation) — no second launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cmath>
#include <cstring>
#include <mutex>

#include "l4_device.cuh"
#include "l4_internal.h"

namespace l4 {
namespace {

constexpr int kPage = 16;
constexpr int kHeadDim = 128;
constexpr int kConsumerWarps = 4;
constexpr int kConsumerThreads = kConsumerWarps * 32;
constexpr int kThreads = kConsumerThreads + 32;      // + 1 producer warp = 160
constexpr int kSliceBytes = kPage * kHeadDim * 2;     // one (page, kv head) K or V slice = 4 KB
constexpr int kHalfBytes = kSliceBytes / 2;           // 16 rows x 64 bf16 (128 B swizzle span)
constexpr int kStageBytes = 2 * kSliceBytes;          // K, V
constexpr int kItemSlots = 4;
constexpr int kMaxG = 8;
constexpr int kMergeStride = kHeadDim + 4;            // floats per head row (bank-conflict padding)
constexpr int kMaxSplits = 512;                       // per (request, kv head)
constexpr int kCombineGroup = 16;                     // two-level combine: splits per group
constexpr int kMaxCombine = kMaxSplits / kCombineGroup;  // partials read by one combine (>= group)
constexpr int kMinChunk = 8;                          // pages
#ifndef L4_ITEMS_PER_CTA
#define L4_ITEMS_PER_CTA 8
#endif
constexpr int kItemsPerCta = L4_ITEMS_PER_CTA;        // automatic chunk target
#ifndef L4_ITEMS_PER_CTA_ALL_SPLIT
#define L4_ITEMS_PER_CTA_ALL_SPLIT 12
#endif
constexpr int kItemsPerCtaAllSplit = L4_ITEMS_PER_CTA_ALL_SPLIT;  // ... when every request is split
constexpr int kAllSplitMinChunk = 128;  // ... and the default chunk has at least this many pages
constexpr int kChunkCands = 16;         // chunk candidates of a large all-split batch
#ifndef L4_CHUNK_SEARCH
#define L4_CHUNK_SEARCH 1
#endif
constexpr int kNoSplitFactor = 2;                     // requests of <= 2C pages are never split
constexpr int kMaxBatch = 8192;
constexpr int kPlanThreads = 1024;
constexpr int kNumBins = 32;
// Warp-item ("quad") units: unsplit items of at most 2^kQuadBin - 1 pages are scheduled four at
// a time, one whole item per consumer warp (no cross-warp merge, no CTA barrier per item).
// 0 disables them.  G <= 4: the four items' Q rows sit in the unit slot; G = 8: each consumer
// warp loads its item's Q rows from global memory into its mma fragments.
#ifndef L4_QUAD_BIN
#define L4_QUAD_BIN 6
#endif
#ifndef L4_PREFETCH_INPUTS
#define L4_PREFETCH_INPUTS 1
#endif
constexpr int kQuadBin = L4_QUAD_BIN;
static_assert(kQuadBin >= 0 && kQuadBin <= 6, "quad items hold at most 63 page ids (two per lane)");
constexpr int kQuadMaxG = 4;
constexpr int kQuad = 4;  // items per quad unit = consumer warps
#ifndef L4_QUAD_TAIL
#define L4_QUAD_TAIL 0
#endif
constexpr int kQuadTailPerCta = L4_QUAD_TAIL;  // CTA-wide items per CTA at the end of the quad suffix
#ifndef L4_QUAD_MIN
#define L4_QUAD_MIN 4
#endif
constexpr int kQuadMinPerCta = L4_QUAD_MIN;  // quads only if there are at least this many per CTA
constexpr int kQuadPagesPerUnitCta = 10;       // ... or q_pages / 10 if fewer (>= 1 per CTA)
constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;

struct __align__(16) WorkItem {
  int b, h, pbeg, pend, last_valid, part_base, nsplit, split;
};
static_assert(sizeof(WorkItem) == 32, "WorkItem is 32 bytes");

#ifdef L4_TRACE
// Development-only timeline probe (scripts/trace_fused.py): %globaltimer at fixed points of
// every CTA, built only into trace variants (scripts/build_variant.sh ... -DL4_TRACE).
__device__ unsigned long long g_trace[4096 * 16];
__device__ unsigned long long g_trace_last[4096 * 4];  // last CTA-wide item: start, pages, splits, index
__device__ __forceinline__ void trace_mark(int k) {  // globaltimer: 256 ns granularity on this part
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_trace[blockIdx.x * 16 + k] = t;
}
#define L4_MARK(k) trace_mark(k)
__device__ __forceinline__ unsigned long long trace_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// accumulated per-CTA counters in slots 12..15 (consumer warp 0 / producer lane 0)
// accumulated in a per-thread register array (tr_acc), stored once when the thread finishes
#define L4_TRACE_ACC unsigned long long tr_acc[16] = {0};
#define trace_add(k, v) (tr_acc[(k)] += (v))
#define L4_TRACE_FLUSH(k) (g_trace[blockIdx.x * 16 + (k)] = tr_acc[(k)])
#else
#define L4_MARK(k) ((void)0)
#endif

#ifdef L4_DEBUG_CKS
// Development-only data checksums per work item (scripts/flake_split.py --cks): XOR of the K and
// V fragments the consumers loaded, XOR of the Q fragments, weighted sum of the page ids the
// producer issued, built only into debug variants (-DL4_DEBUG_CKS).
__device__ unsigned g_cks[16384 * 4];
#endif

// Header region (256 B): plan summary + dynamic scheduler state.
struct __align__(16) PlanHeader {
  int n_items, chunk, num_ctas, max_splits;
  int batch, num_kv_heads, items_cap, n_wide;  // n_wide: items before the quad units
  int tail_requests, tail_chunk, quad_pages, pad2[5];  // quad_pages: see plan_core's QPages_out
  int sched_next, sched_done, pad3[14];  // ticket counter and finished-CTA count (self-resetting)
};
static_assert(sizeof(PlanHeader) == 128, "PlanHeader is 128 bytes");

// ------------------------------------------------------------------ workspace layout
struct WsLayout {
  size_t header, counters, gcount, items, part_lse, part_o, total;
  int items_cap;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

WsLayout ws_layout(int B, int Hkv, int G, int items_cap) {
  WsLayout L;
  L.items_cap = items_cap;
  L.header = 0;
  L.counters = 256;
  // counters are self-cleaning across runs, so their region must not depend on B: a workspace
  // reused with another batch size never sees stale items where its counters are
  (void)B;
  L.gcount = align256(L.counters + (size_t)kMaxBatch * Hkv * sizeof(int));  // group counters, one per slot
  L.items = align256(L.gcount + (size_t)items_cap * sizeof(int));
  L.part_lse = align256(L.items + (size_t)items_cap * sizeof(WorkItem));
  L.part_o = align256(L.part_lse + (size_t)items_cap * G * sizeof(float));
  L.total = align256(L.part_o + (size_t)items_cap * G * kHeadDim * sizeof(float));
  return L;
}

// The layout is a pure function of (Hkv, G, workspace_bytes): plan and run
// both derive the largest item capacity that fits the caller's workspace.
bool ws_layout_from_bytes(int B, int Hkv, int G, size_t bytes, WsLayout* out) {
  const WsLayout z = ws_layout(B, Hkv, G, 0);
  if (bytes < z.total) return false;
  const size_t per_item =
      sizeof(int) + sizeof(WorkItem) + (size_t)G * sizeof(float) + (size_t)G * kHeadDim * sizeof(float);
  int64_t cap = (int64_t)((bytes - z.total) / per_item);
  cap = std::min<int64_t>(cap, INT_MAX / 64);
  while (cap > 0 && ws_layout(B, Hkv, G, (int)cap).total > bytes) --cap;
  if (cap <= 0) return false;
  *out = ws_layout(B, Hkv, G, (int)cap);
  return true;
}

l4_status get_device(int* dev_out) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) {
    set_error("cudaGetDevice failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  *dev_out = dev;
  return L4_OK;
}

// ------------------------------------------------------------------ parameter checks
l4_status check_params(const l4_decode_params* p, int* G_out) {
  L4_CHECK_ARG(p != nullptr, "decode params is NULL");
  L4_CHECK_ARG(p->batch >= 0, "batch must be >= 0");
  if (p->batch > kMaxBatch) return fail(L4_ERR_UNSUPPORTED, "batch > 8192 is not supported");
  L4_CHECK_ARG(p->num_q_heads >= 1 && p->num_kv_heads >= 1, "head counts must be >= 1");
  L4_CHECK_ARG(p->num_q_heads % p->num_kv_heads == 0, "num_q_heads must be a multiple of num_kv_heads");
  if (p->head_dim != kHeadDim) return fail(L4_ERR_UNSUPPORTED, "head_dim must be 128");
  if (p->page_size != kPage) return fail(L4_ERR_UNSUPPORTED, "page_size must be 16");
  const int G = p->num_q_heads / p->num_kv_heads;
  if (!(G == 1 || G == 2 || G == 4 || G == 8)) return fail(L4_ERR_UNSUPPORTED, "GQA group must be 1, 2, 4 or 8");
  L4_CHECK_ARG(p->out_dtype == L4_DT_F32 || p->out_dtype == L4_DT_BF16, "out_dtype must be F32 or BF16");
  L4_CHECK_ARG(std::isfinite(p->sm_scale), "sm_scale must be finite");
  L4_CHECK_ARG((p->flags & ~(L4_DECODE_EARLY_INPUTS | L4_DECODE_EARLY_PLAN)) == 0, "unknown decode flags");
  *G_out = G;
  return L4_OK;
}

int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Upper bound on work items for any batch with <= max_total_pages pages.
int items_cap_for(const l4_decode_params* p, int64_t max_total_pages, int num_ctas) {
  const int64_t B = p->batch, Hkv = p->num_kv_heads;
  int64_t cap;
  if (p->chunk_pages < 0) {
    cap = B * Hkv;
  } else if (p->chunk_pages > 0) {
    cap = Hkv * (B + ceil_div64(max_total_pages, p->chunk_pages));
  } else {
    // C >= T*Hkv/(W*k) => Hkv * sum ceil(p_b / C) <= W*k + Hkv*B (k: the larger chunk target)
    cap = std::min(Hkv * (B + ceil_div64(max_total_pages, kMinChunk)),
                   Hkv * B + (int64_t)num_ctas * std::max(kItemsPerCta, kItemsPerCtaAllSplit) + Hkv);
  }
  cap = std::max<int64_t>(cap, 1);
  return (int)std::min<int64_t>(cap, INT_MAX / 64);
}

// =================================================================== a1: planner
struct PlanArgs {
  const int* kv_len;
  const int* indptr;
  int B, Hkv, num_ctas, forced_chunk, items_cap, quad_bin;
  PlanHeader* header;
  WorkItem* items;
  int* counters;
};

constexpr int kPlanMaxWarps = kPlanThreads / 32;

// Block-wide (sum int64, max int, min int, or bits) in one pass.
__device__ void block_reduce4(long long v, int m, int mn, unsigned bits, long long* s_ll, int* s_i, int* s_mn,
                              unsigned* s_u, long long* sum_out, int* max_out, int* min_out, unsigned* or_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    bits |= __shfl_xor_sync(0xffffffffu, bits, o);
  }
  __syncthreads();
  if (lane == 0) {
    s_ll[warp] = v;
    s_i[warp] = m;
    s_mn[warp] = mn;
    s_u[warp] = bits;
  }
  __syncthreads();
  long long t = 0;
  int mm = 0, mi = INT_MAX;
  unsigned bb = 0;
#pragma unroll 8
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
    t += s_ll[i];
    mm = max(mm, s_i[i]);
    mi = min(mi, s_mn[i]);
    bb |= s_u[i];
  }
  *sum_out = t;
  *max_out = mm;
  *min_out = mi;
  *or_out = bb;
}

__device__ __forceinline__ int pages_of(int L) { return L > 0 ? (L + kPage - 1) / kPage : 0; }

__device__ __forceinline__ int nsplit_of(int pages, int C) {
  if (pages <= kNoSplitFactor * C) return 1;  // also pages == 0
  return (pages + C - 1) / C;
}

__device__ __forceinline__ int bin_of(int pages, int nsplit) {
  if (pages <= 0) return 0;
  const int ip = nsplit == 1 ? pages : (pages + nsplit - 1) / nsplit;  // pages of the largest split
  return min(kNumBins - 1, 32 - __clz(ip));      // bit_length(ip)
}

// Chunk choice of a large all-split batch (plan_core, §4.1): among kChunkCands chunks from c12 (12
// items per CTA) to 1.3x the default chunk c8, the one whose last round of items is closest to 85%
// full (ties: the larger chunk).  Block-wide (every thread calls it); s_cand aliases s_wcnt, which
// it leaves zeroed.  Kept out of line: inlined, its unrolled code cost mixed batches 0.3-0.5%
// (measured with it compiled out), although they never execute it.
__device__ __noinline__ long long chunk_search(const int* s_len, int B, int Hkv, int num_ctas, int items_cap,
                                               int Pmax, long long c8, long long c12, long long* s_cand,
                                               int* s_wcnt) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nw = nthr >> 5;
  long long Cl = c8;
  const long long c_lo = max(c12, (long long)((Pmax + kMaxSplits - 1) / kMaxSplits));
  const long long c_hi = c8 + c8 * 3 / 10;
  long long cand[kChunkCands];
  unsigned cnt[kChunkCands];
#pragma unroll
  for (int k = 0; k < kChunkCands; ++k) {
    cand[k] = c_lo + (c_hi - c_lo) * k / (kChunkCands - 1);
    cnt[k] = 0;
  }
  for (int b = tid; b < B; b += nthr) {
    const unsigned pg = (unsigned)pages_of(s_len[b]);
#pragma unroll
    for (int k = 0; k < kChunkCands; ++k) {
      const unsigned c = (unsigned)cand[k];  // < 2^30 (chunks are capped at INT_MAX / 4)
      cnt[k] += pg <= kNoSplitFactor * c ? 1u : (pg + c - 1) / c;
    }
  }
#pragma unroll
  for (int k = 0; k < kChunkCands; ++k) {
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt[k] += __shfl_xor_sync(0xffffffffu, cnt[k], o);
    if (lane == 0) s_cand[warp * kChunkCands + k] = (long long)cnt[k];
  }
  __syncthreads();
  double best = 2.0;
#pragma unroll
  for (int k = 0; k < kChunkCands; ++k) {
    long long n = 0;
    for (int w = 0; w < nw; ++w) n += s_cand[w * kChunkCands + k];
    n *= Hkv;
    const double frac = (double)(n % num_ctas) / num_ctas;
    const double score = fabs(frac - 0.85);
    if (n <= items_cap && score <= best) {  // ties: the later (larger) chunk
      best = score;
      Cl = cand[k];
    }
  }
  __syncthreads();  // every thread read s_cand: give s_wcnt back to pass 1, zeroed
  for (int x = tid; x < nw * kNumBins; x += nthr) s_wcnt[x] = 0;
  __syncthreads();
  return Cl;
}

// Shared-memory scratch of plan_core (bytes; 8-byte aligned base).
constexpr int kPlanScratchBytes = 32 * 8 + 36 * 4 + 32 * 4 + 32 * 4 + kPlanMaxWarps * kNumBins * 4 + 32 * 4 + 32 * 4;

// The planner (a1), run by every thread of a CTA: reads kv_len / indptr, chooses the chunk C,
// and orders the requests by length bin, longest bin first, request index ascending inside a
// bin (deterministic).  Leaves in shared memory: s_len / s_ptr [B] (kv_len, indptr), s_rb [B]
// (request at rank r | its split count << 16), s_off [B+1] (first item of rank r; rank r owns nsplit * Hkv items,
// contiguous per kv head), and returns C, the item count N and the largest page count.
// Used by plan_kernel (materialised work list) and by the fused decode kernel (every CTA
// plans redundantly in its own shared memory: no planner launch, no global work list).
// Ranking is warp-blocked (warp w owns a contiguous range of requests): ~10 block barriers
// whatever B is.
__device__ void plan_core(const int* __restrict__ kv_len, const int* __restrict__ indptr, int B, int Hkv,
                          int num_ctas, int forced_chunk, int items_cap, int* s_len, int* s_ptr, int* s_rb,
                          int* s_off, unsigned char* scratch, int* C_out, int* N_out, int* Pmax_out,
                          int quad_bin, int* Wide_out, int* QPages_out, int* TailChunk_out = nullptr) {
  long long* s_ll = reinterpret_cast<long long*>(scratch);
  int* s_i = reinterpret_cast<int*>(scratch + 32 * 8);
  unsigned* s_u = reinterpret_cast<unsigned*>(scratch + 32 * 8 + 36 * 4);
  int* s_w = reinterpret_cast<int*>(scratch + 32 * 8 + 36 * 4 + 32 * 4);        // per-warp sums
  int* s_wcnt = reinterpret_cast<int*>(scratch + 32 * 8 + 36 * 4 + 32 * 4 + 32 * 4);  // [nw][kNumBins]
  int* s_ms = s_wcnt + kPlanMaxWarps * kNumBins;  // per-warp lowest bin of a split request
  int* s_mn = s_ms + 32;                           // per-warp smallest page count
  // [nw][kChunkCands] item counts of the chunk search: aliases the per-warp bin counts s_wcnt
  // (same size), which are re-zeroed after the search
  long long* s_cand = reinterpret_cast<long long*>(s_wcnt);
  static_assert(kChunkCands * 8 == kNumBins * 4, "s_cand aliases s_wcnt");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nw = nthr >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  long long T;
  int Pmax, Pmin;
  unsigned bins_seen;  // bit k: some request's unsplit bin (bit_length of its pages) is k
  {
    long long sum = 0;
    int mx = 0, mn = INT_MAX;
    unsigned seen = 0u;
    auto take = [&](int b, int Lv, int Pv) {
      s_len[b] = Lv;
      s_ptr[b] = Pv;
      const int pg = pages_of(Lv);
      sum += pg;
      mx = max(mx, pg);
      mn = min(mn, pg);
      seen |= 1u << bin_of(pg, 1);
    };
    // one round of loads: 16-byte vectors of both arrays (B <= 1024 needs <= 2 per thread at
    // 160 threads), scalars for the ragged tail or unaligned arrays
    const bool vec = ((reinterpret_cast<uintptr_t>(kv_len) | reinterpret_cast<uintptr_t>(indptr)) & 15u) == 0;
    const int B4 = vec ? (B >> 2) : 0;
    for (int v0 = tid; v0 < B4; v0 += 2 * nthr) {
      int4 Lv[2], Pv[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int v = v0 + u * nthr;
        Lv[u] = v < B4 ? reinterpret_cast<const int4*>(kv_len)[v] : make_int4(0, 0, 0, 0);
        Pv[u] = v < B4 ? reinterpret_cast<const int4*>(indptr)[v] : make_int4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int v = v0 + u * nthr;
        if (v < B4) {
          take(4 * v, Lv[u].x, Pv[u].x);
          take(4 * v + 1, Lv[u].y, Pv[u].y);
          take(4 * v + 2, Lv[u].z, Pv[u].z);
          take(4 * v + 3, Lv[u].w, Pv[u].w);
        }
      }
    }
    for (int b0 = 4 * B4 + tid; b0 < B; b0 += 4 * nthr) {  // four loads of each array in flight
      int Lv[4], Pv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b = b0 + u * nthr;
        Lv[u] = b < B ? kv_len[b] : 0;
        Pv[u] = b < B ? indptr[b] : 0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b = b0 + u * nthr;
        if (b < B) take(b, Lv[u], Pv[u]);
      }
    }
    for (int x = tid; x < nw * kNumBins; x += nthr) s_wcnt[x] = 0;
    block_reduce4(sum, mx, mn, seen, s_ll, s_i, s_mn, s_u, &T, &Pmax, &Pmin, &bins_seen);  // its barriers publish s_len/s_ptr
  }
  if (tid == 0) L4_MARK(6);
  // chunk size C (pages per work item)
  long long Cl;
  if (forced_chunk > 0) {
    Cl = forced_chunk;
  } else if (forced_chunk < 0) {
    Cl = INT_MAX / 4;
  } else {
    // 32-bit division when it fits (a 64-bit one is a long software sequence on the critical path)
    auto chunk_for = [&](int items_per_cta) -> long long {
      const long long denom = (long long)num_ctas * items_per_cta;
      const long long num = T * Hkv + denom - 1;
      const long long q = num < (1ll << 31) ? (long long)((unsigned)num / (unsigned)denom) : num / denom;
      return max((long long)kMinChunk, q);
    };
    Cl = chunk_for(kItemsPerCta);
    // A large batch whose every request is split (a long-context batch: C4, an L4 long-range
    // stage) has no short unsplit items to fill the end of the launch, so how full its last round
    // of items is decides its tail: with N items over W CTAs, a last round that only a few CTAs
    // enter (N / W just above an integer) leaves the rest idle for a whole item, and one that
    // most CTAs enter evens out their progress spread.  Measured (plain calls, forced chunks):
    // C4 1544-1563 us when frac(N / W) is 0.73-0.97, 1566-1570 at 0.3-0.4, 1578-1601 at
    // 0.03-0.22; 25 x 39454 tokens 570 us at 0.78-0.81 vs 584-587 at 0.11-0.16; 12 x 84547 587
    // at 0.84 vs 606-608 at 0.08-0.11.  So among chunks from the 12-items-per-CTA chunk up to
    // 1.3x the default one the planner takes the chunk whose last round is closest to 85% full
    // (ties: the larger chunk, fewer combines).  A/B against a fixed 12 items per CTA (same box):
    // C4 1588 -> 1571 us, 25 x 39454 591 -> 586, 64 x 16384 623 -> 619, 12 x 84547 and 8 x 131072
    // unchanged.  Small all-split batches (default chunk < kAllSplitMinChunk pages) are combine-
    // and latency-bound and keep the default.
    if (L4_CHUNK_SEARCH && B > 0 && Cl >= kAllSplitMinChunk && (long long)Pmin > kNoSplitFactor * Cl)
      Cl = chunk_search(s_len, B, Hkv, num_ctas, items_cap, Pmax, Cl, chunk_for(kItemsPerCtaAllSplit), s_cand, s_wcnt);
  }
  Cl = max(Cl, (long long)((Pmax + kMaxSplits - 1) / kMaxSplits));
  int C = (int)min(Cl, (long long)(INT_MAX / 4));
  if (__popc(bins_seen) <= 1 && Pmax <= kNoSplitFactor * C && (long long)B * Hkv <= items_cap) {
    // Fast path (same plan bit for bit): no request is split and all fall in one length bin (a
    // homogeneous batch, or an L4 stage whose range lies within one power-of-two bucket), so the
    // stable rank order is the request order and rank r owns items [r Hkv, (r + 1) Hkv): no
    // histogram, scatter or scan (~2.5 us of block barriers and shared-memory passes at B = 1024).
    for (int b = tid; b < B; b += nthr) s_rb[b] = b | (1 << 16);
    for (int r = tid; r <= B; r += nthr) s_off[r] = r * Hkv;
    const int bin = bins_seen ? __ffs(bins_seen) - 1 : 0;
    const bool has_quads = quad_bin > 0 && bin <= quad_bin && B > 0;
    __syncthreads();
    if (TailChunk_out) *TailChunk_out = 0;
    *C_out = C;
    *N_out = B * Hkv;
    *Pmax_out = Pmax;
    *Wide_out = has_quads ? 0 : B * Hkv;
    *QPages_out = has_quads ? pages_of(s_len[0]) : 0;
    return;
  }
  // ---- ranks: counting sort by bin (descending), stable in request order.  Warp w owns the
  // contiguous request range [r0, r1); pass 1 also counts the items, so growing C when the
  // work list does not fit the workspace repeats pass 1 only (block-uniform loop).
  const int tiles = (B + 31) >> 5;
  const int tpw = (tiles + nw - 1) / nw;
  const int r0 = min(B, warp * tpw * 32), r1 = min(B, r0 + tpw * 32);
  long long N;
  int min_split_bin;
  for (;;) {
    int wsum = 0, wms = kNumBins;
    // pass 1: per-warp bin histogram + item count, tile by tile (a version that issued the shared
    // loads of 8 tiles together measured the same: random-composition sweep, scripts/gpu_run35.sh)
    for (int t0 = r0; t0 < r1; t0 += 32) {
      const int b = t0 + lane;
      int bin = -1;
      if (b < r1) {
        const int pg = pages_of(s_len[b]);
        const int ns = nsplit_of(pg, C);
        bin = bin_of(pg, ns);
        wsum += ns;
        if (ns > 1) wms = min(wms, bin);
        s_off[b] = bin | (ns << 16);  // kept for pass 2 (s_off is free until the scan)
      }
      // one shared atomic per distinct bin of the tile (counts only: tiles independent; per-lane
      // atomics serialise on a tile of equal bins: B = 128 short requests 45.0 -> 43.4 us)
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      if (bin >= 0 && (peers & lt_mask) == 0) atomicAdd(&s_wcnt[warp * kNumBins + bin], __popc(peers));
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
      wms = min(wms, __shfl_xor_sync(0xffffffffu, wms, o));
    }
    if (lane == 0) {
      s_w[warp] = wsum;  // not s_i: slower warps may still read block_reduce4's s_i
      s_ms[warp] = wms;
    }
    __syncthreads();
    N = 0;
    min_split_bin = kNumBins;
    for (int w = 0; w < nw; ++w) {
      N += s_w[w];
      min_split_bin = min(min_split_bin, s_ms[w]);
    }
    N *= Hkv;
    if (N <= items_cap || C >= INT_MAX / 8) break;
    C *= 2;
    for (int x = tid; x < nw * kNumBins; x += nthr) s_wcnt[x] = 0;
    __syncthreads();
  }
  if (tid == 0) L4_MARK(7);
  // Quad bins: every item of bins <= quad_bin must be unsplit, so the quad bins end below the
  // lowest bin that holds a split request (a split request's largest split has more than 2C/3
  // pages, so this never cuts below bit_length(floor(2C/3) + 1) - 1).
  if (quad_bin > 0) quad_bin = min(quad_bin, min_split_bin - 1);
  if (warp == 0) {  // bases: bins in descending order, then warps in request order
    const int bin = kNumBins - 1 - lane;
    int tot = 0;
    for (int w = 0; w < nw; ++w) tot += s_wcnt[w * kNumBins + bin];
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    int base = incl - tot;
    if (bin == quad_bin) s_i[34] = base;  // first rank of the quad bins (bins <= quad_bin)
    const unsigned used = __ballot_sync(0xffffffffu, tot > 0);
    if (lane == 0) s_i[33] = __popc(used) <= 1;  // one bin: the rank order is the request order
    for (int w = 0; w < nw; ++w) {
      const int c = s_wcnt[w * kNumBins + bin];
      s_wcnt[w * kNumBins + bin] = base;
      base += c;
    }
  }
  __syncthreads();
  // read before the barriers below: the scratch is the merge area, which consumers overwrite
  // once their first item is done
  const int quad_rank = s_i[34];
  const bool one_bin = s_i[33] != 0;
  if (tid == 0) L4_MARK(8);
  if (one_bin) {  // fast path, same result: a stable sort of one bin is the identity
    for (int b = tid; b < B; b += nthr) s_rb[b] = b | ((s_off[b] >> 16) << 16);
  } else {
    for (int t0 = r0; t0 < r1; t0 += 32) {  // pass 2: scatter (request | nsplit << 16) to its rank
      const int b = t0 + lane;
      int bin = -1, ns = 0;
      if (b < r1) {
        const int packed = s_off[b];                // pass 1's (bin, nsplit)
        bin = packed & 0xffff;
        ns = packed >> 16;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, bin);
      const int lower = __popc(peers & lt_mask);
      int pos = 0;
      if (bin >= 0) pos = s_wcnt[warp * kNumBins + bin] + lower;
      __syncwarp();
      if (bin >= 0) {
        s_rb[pos] = b | (ns << 16);  // b < 8192, ns <= kMaxSplits
        if (lower == 0) s_wcnt[warp * kNumBins + bin] += __popc(peers);
      }
      __syncwarp();
    }
  }
  __syncthreads();
  if (tid == 0) L4_MARK(9);
  // ---- item offsets: exclusive scan of nsplit * Hkv in rank order (same warp ranges); with no
  // split request (N = B * Hkv) it is r * Hkv (fast path, same result)
  if (N == (long long)B * Hkv) {
    for (int r = tid; r <= B; r += nthr) s_off[r] = r * Hkv;
  } else {
    int wsum = 0;
    for (int t0 = r0; t0 < r1; t0 += 32) {
      const int r = t0 + lane;
      wsum += r < r1 ? (s_rb[r] >> 16) : 0;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) wsum += __shfl_xor_sync(0xffffffffu, wsum, o);
    if (lane == 0) s_w[warp] = wsum;  // pass 1's counts in s_w were read two barriers ago
    __syncthreads();
    int carry = 0;
    for (int w = 0; w < warp; ++w) carry += s_w[w];
    carry *= Hkv;
    for (int t0 = r0; t0 < r1; t0 += 32) {
      const int r = t0 + lane;
      const int cnt = r < r1 ? (s_rb[r] >> 16) * Hkv : 0;
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (r < r1) s_off[r] = carry + incl - cnt;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (tid == 0) s_off[B] = (int)N;
  }
  __syncthreads();
  if (TailChunk_out) *TailChunk_out = 0;  // no guided tail (DESIGN §4.2 negative results)
  *C_out = C;
  *N_out = (int)N;
  *Pmax_out = Pmax;
  // items before the first quad-bin rank run CTA-wide; the rest are grouped four per unit
  const bool has_quads = quad_bin > 0 && quad_rank < B;
  *Wide_out = has_quads ? s_off[quad_rank] : (int)N;
  // pages of the first quad-eligible request (its bin is the largest; within a bin, < 2x more)
  *QPages_out = has_quads ? pages_of(s_len[s_rb[quad_rank] & 0xffff]) : 0;
}

// Work item `i` of the plan held in shared memory (fused path) — the same item plan_kernel
// writes at index i: rank r = the last rank whose first item is <= i, then (kv head, split).
__device__ __forceinline__ WorkItem item_from_plan(int i, int n, const int* s_len, const int* s_ptr,
                                                   const int* s_rb, const int* s_off, int B, int Hkv) {
  WorkItem it;
  if (i >= n) {
    it.b = -1; it.h = 0; it.pbeg = 0; it.pend = 0; it.last_valid = 0; it.part_base = 0; it.nsplit = 1; it.split = 0;
    return it;
  }
  int lo = 0;
  if (n == B * Hkv) {  // no split request: rank r owns items [r * Hkv, (r + 1) * Hkv)
    lo = i / Hkv;
  } else {
    int hi = B - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= i) lo = mid; else hi = mid - 1;
    }
  }
  const int b = s_rb[lo] & 0xffff, ns = s_rb[lo] >> 16;
  const int L = s_len[b];
  const int pg = pages_of(L);
  const int loc = i - s_off[lo];
  const int h = loc / ns, sp = loc - h * ns;
  const int p0 = (sp * pg) / ns, p1 = ((sp + 1) * pg) / ns;
  it.b = b;
  it.h = h;
  it.pbeg = s_ptr[b] + p0;
  it.pend = s_ptr[b] + p1;
  it.last_valid = p1 == pg ? (pg > 0 ? L - (pg - 1) * kPage : 0) : kPage;
  it.part_base = s_off[lo] + h * ns;
  it.nsplit = ns;
  it.split = sp;
  return it;
}

// Materialised plan: one CTA (<= 1024 threads) runs plan_core and writes the work list,
// so one plan serves many l4_decode_run calls (e.g. every layer of a decode iteration).
__global__ void __launch_bounds__(kPlanThreads, 1) plan_kernel(PlanArgs a) {
  // PDL: let the dependent decode kernel start its prologue now; it waits
  // (griddepcontrol.wait) for this grid's completion before reading the plan.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(16) unsigned char plan_smem_raw[];
  const int Bs = max(a.B, 1);
  unsigned char* scratch = plan_smem_raw;
  int* s_len = reinterpret_cast<int*>(plan_smem_raw + kPlanScratchBytes);
  int* s_ptr = s_len + Bs;
  int* s_rb = s_ptr + Bs;
  int* s_off = s_rb + Bs;
  const int tid = threadIdx.x, nthr = blockDim.x;
  int C, N, Pmax, Nw, Qb, Ct;
  plan_core(a.kv_len, a.indptr, a.B, a.Hkv, a.num_ctas, a.forced_chunk, a.items_cap, s_len, s_ptr, s_rb, s_off,
            scratch, &C, &N, &Pmax, a.quad_bin, &Nw, &Qb, &Ct);
  // ---- items: one thread per (request rank, kv head) writes that pair's splits
  for (int x = tid; x < a.B * a.Hkv; x += nthr) {
    const int r = x / a.Hkv, h = x - r * a.Hkv;
    const int b = s_rb[r] & 0xffff, ns = s_rb[r] >> 16;
    const int L = s_len[b];
    const int pg = pages_of(L);
    const int first = s_off[r] + h * ns;
    const int pbase = s_ptr[b];
    const int last_valid = pg > 0 ? L - (pg - 1) * kPage : 0;
    int p0 = 0;
    for (int sp = 0; sp < ns; ++sp) {
      const int p1 = ((sp + 1) * pg) / ns;  // pg * ns < 2^31 (ns <= 512)
      int4* dst = reinterpret_cast<int4*>(a.items + first + sp);
      dst[0] = make_int4(b, h, pbase + p0, pbase + p1);
      dst[1] = make_int4(p1 == pg ? last_valid : kPage, first, ns, sp);
      p0 = p1;
    }
  }
  for (int x = tid; x < a.B * a.Hkv; x += nthr) a.counters[x] = 0;
  if (tid == 0) {
    PlanHeader hd;
    memset(&hd, 0, sizeof(hd));
    hd.n_items = N;
    hd.chunk = C;
    hd.num_ctas = a.num_ctas;
    hd.max_splits = nsplit_of(Pmax, C);
    hd.batch = a.B;
    hd.num_kv_heads = a.Hkv;
    hd.items_cap = a.items_cap;
    hd.n_wide = Nw;
    hd.quad_pages = Qb;
    hd.tail_chunk = Ct;  // guided tail chunk (0: none)
    hd.sched_next = 0;
    hd.sched_done = 0;
    *a.header = hd;
  }
}

// =================================================================== a2 + a3: split-KV kernel
struct RunArgs {
  const __nv_bfloat16* q;
  void* out;
  float* lse;
  const int* indices;
  const WorkItem* items;
  PlanHeader* header;
  int* counters;
  int* gcount;
  float* part_o;
  float* part_lse;
  int Hq, Hkv;
  float scale_log2;  // sm_scale * log2(e)
  int out_bf16;
  // fused path only: the planner's inputs (every CTA plans in shared memory)
  const int* kv_len;
  const int* indptr;
  int B, forced_chunk, items_cap;
  int quad_bin;  // kQuadBin (0: no quad units)
  int early;  // 1: L4_DECODE_EARLY_INPUTS, 2: L4_DECODE_EARLY_PLAN (fused path), 0: neither
  long long n_indices;  // page_indices entries (fused path; 0: unknown, no prefetch)
};

struct __align__(16) SlotItem {  // unit handed from the producer to the consumers
  WorkItem it[kQuad];  // CTA-wide unit: it[0]; quad unit: one item per consumer warp
  int idx;             // work-item index of it[0] (partial slot of a split item)
  int nsub;            // 0: CTA-wide unit (it[0].b < 0: no more work); 1..4: quad unit
  int maxnp, pad;      // quad: pages of its longest item
};

constexpr int kCombineScratchBytes = (kMaxCombine * kMaxG + 2 * kMaxG) * 4 + kConsumerThreads * 16;
constexpr int cmax(int x, int y) { return x > y ? x : y; }
constexpr int align16c(int x) { return (x + 15) & ~15; }

// Shared memory of decode_kernel<G>, sized for its GQA group (Q slots of G rows, a warp merge
// area of G heads that doubles as planner / combine scratch).  The page ring must cover HBM
// latency x the CTA's share of the bandwidth plus the consumers' per-item epilogue: 8 stages.
// A depth that is not a multiple of the 4 consumer warps needs stage sequence numbers: pages go
// to warps round-robin inside an item, so the previous use of a stage may belong to another,
// lagging warp and still be in flight, and a parity-only wait would return on the older phase;
// with `seq` the consumer of page q first waits until the producer armed the stage for q.  With
// 8 stages page q - 8 was consumed by the same warp (or before the item barrier), so the check is
// compiled out.  (Measured: 10 stages + seq for G <= 4 changed C2/C3/C4 by -1..+1% and small
// batches by +2%; not kept.)
#ifndef L4_STAGES_SMALL_G
#define L4_STAGES_SMALL_G 8
#endif
template <int G>
struct SmemLayout {
  static constexpr int stages_n = G == 8 ? 8 : L4_STAGES_SMALL_G;
  static constexpr bool quads = kQuadBin > 0;
  // G <= 4: a unit slot holds the Q rows of four items (+12 KB at G = 4); G = 8: four items' Q
  // rows would not fit 2 CTAs/SM (+24 KB), so each consumer warp loads its quad item's rows from
  // global memory straight into its mma fragments
  static constexpr bool q_global = G > kQuadMaxG;
  static constexpr int qslot_bytes = (quads && !q_global ? kQuad : 1) * G * kHeadDim * 2;  // Q rows of one unit
  static constexpr int merge_bytes =
      align16c(cmax(kConsumerWarps * G * kMergeStride * 4, cmax(kPlanScratchBytes, kCombineScratchBytes)));
  static constexpr int stages = 0;
  static constexpr int qslots = stages + stages_n * kStageBytes;
  static constexpr int items = align16c(qslots + kItemSlots * qslot_bytes);
  static constexpr int merge_o = items + kItemSlots * (int)sizeof(SlotItem);
  static constexpr int merge_m = merge_o + merge_bytes;
  static constexpr int merge_l = merge_m + kConsumerWarps * kMaxG * 4;
  static constexpr int bars = merge_l + kConsumerWarps * kMaxG * 4;
  static constexpr int nbars = 2 * stages_n + 2 * kItemSlots;
  static constexpr int seq = bars + nbars * 8;  // int [stages_n]: page sequence number armed per stage
  static constexpr int flag = seq + stages_n * 4;
  static constexpr int total = align16c(flag + 16);
  static constexpr int alloc = total + 1024;  // room to align the base to 1024 B (128B swizzle)
  static_assert(merge_o % 16 == 0 && total % 16 == 0 && bars % 8 == 0, "aligned areas");
};
// Fused path: plan arrays s_len, s_ptr, s_rb [B] and s_off [B+1] after the kernel's own layout.
inline size_t fused_plan_bytes(int B) { return ((size_t)(4 * B + 1) * 4 + 15) & ~size_t(15); }
constexpr int kFusedMaxBatch = 1024;  // 2 CTAs per SM still fit (2 x <= 111 KB)
static_assert(2 * (SmemLayout<4>::alloc + (4 * kFusedMaxBatch + 1) * 4 + 16 + 1024) <= 228 * 1024, "2 CTAs/SM (G=4)");
static_assert(2 * (SmemLayout<8>::alloc + (4 * kFusedMaxBatch + 1) * 4 + 16 + 1024) <= 228 * 1024, "2 CTAs/SM (G=8)");

__device__ __forceinline__ void store_out(const RunArgs& a, size_t idx, float v) {
  if (a.out_bf16)
    reinterpret_cast<__nv_bfloat16*>(a.out)[idx] = __float2bfloat16_rn(v);
  else
    reinterpret_cast<float*>(a.out)[idx] = v;
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.global.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// a3: log-sum-exp combine (FlashDecoding aggregation) of `cnt` partials held at
// workspace slots slot0, slot0 + stride, ... (normalised O [G][128] and base-2 lse [G] each):
//   M = max_s lse_s,  w_s = 2^(lse_s - M),  O = sum_s w_s O_s / sum_s w_s,  lse = M + log2 sum_s w_s.
// The result goes to the output rows row0 .. row0 + G - 1 (to_output) or back to slot `dst` in
// the same partial form (a group partial of the two-level combine).  Run by the 128 consumer
// threads; float4 loads, up to 8 partials in flight per thread; fixed summation order.
template <int G>
__device__ __forceinline__ void combine_slots(const RunArgs& a, float* scratch, int slot0, int stride, int cnt,
                                              bool to_output, size_t row0, int dst, int ct) {
  using namespace dev;
  const int warp = ct >> 5, lane = ct & 31;
  float* s_w = scratch;                         // [cnt][G]: lse, then weights
  float* s_M = scratch + kMaxCombine * kMaxG;   // [G]
  float* s_L = s_M + kMaxG;                     // [G]
  float4* s_acc = reinterpret_cast<float4*>(s_L + kMaxG);
  for (int x = ct; x < cnt * G; x += kConsumerThreads) {
    const int c = x / G, head = x - c * G;
    s_w[x] = __ldcg(a.part_lse + (size_t)(slot0 + c * stride) * G + head);
  }
  named_bar_sync(1, kConsumerThreads);
  for (int head = warp; head < G; head += kConsumerWarps) {
    float m = -INFINITY;
    for (int c = lane; c < cnt; c += 32) m = fmaxf(m, s_w[c * G + head]);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    const float mu = (m == -INFINITY) ? 0.f : m;
    float l = 0.f;
    for (int c = lane; c < cnt; c += 32) {
      const float w = ex2(s_w[c * G + head] - mu);
      s_w[c * G + head] = w;
      l += w;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
    if (lane == 0) {
      s_M[head] = m;
      s_L[head] = l;
    }
  }
  named_bar_sync(1, kConsumerThreads);
  constexpr int F4 = G * (kHeadDim / 4);                  // float4 per partial
  constexpr int kSpan = F4 < kConsumerThreads ? F4 : kConsumerThreads;
  constexpr int kGroups = kConsumerThreads / kSpan;       // thread groups splitting the partials
  constexpr int kPer = F4 / kSpan;                        // float4 per thread
  const int f0 = ct % kSpan, grp = ct / kSpan;
  float4 acc[kPer];
#pragma unroll
  for (int i = 0; i < kPer; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  int c = grp;
  for (; c + 7 * kGroups < cnt; c += 8 * kGroups) {
    float4 v[8][kPer];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float4* src = reinterpret_cast<const float4*>(a.part_o + (size_t)(slot0 + (c + u * kGroups) * stride) * G * kHeadDim);
#pragma unroll
      for (int i = 0; i < kPer; ++i) v[u][i] = __ldcg(src + f0 + i * kSpan);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < kPer; ++i) {
        const float w = s_w[(c + u * kGroups) * G + (f0 + i * kSpan) / 32];
        acc[i].x += w * v[u][i].x;
        acc[i].y += w * v[u][i].y;
        acc[i].z += w * v[u][i].z;
        acc[i].w += w * v[u][i].w;
      }
  }
  for (; c < cnt; c += kGroups) {
    const float4* src = reinterpret_cast<const float4*>(a.part_o + (size_t)(slot0 + c * stride) * G * kHeadDim);
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const float4 v = __ldcg(src + f0 + i * kSpan);
      const float w = s_w[c * G + (f0 + i * kSpan) / 32];
      acc[i].x += w * v.x;
      acc[i].y += w * v.y;
      acc[i].z += w * v.z;
      acc[i].w += w * v.w;
    }
  }
  if constexpr (kGroups > 1) {  // fold the thread groups in a fixed order
    s_acc[grp * kSpan + f0] = acc[0];
    named_bar_sync(1, kConsumerThreads);
    if (grp == 0) {
      acc[0] = s_acc[f0];
      for (int g2 = 1; g2 < kGroups; ++g2) {
        const float4 t = s_acc[g2 * kSpan + f0];
        acc[0].x += t.x;
        acc[0].y += t.y;
        acc[0].z += t.z;
        acc[0].w += t.w;
      }
    }
  }
  if (grp != 0) return;
#pragma unroll
  for (int i = 0; i < kPer; ++i) {
    const int f = f0 + i * kSpan, head = f / 32, d = (f % 32) * 4;
    const float L = s_L[head], M = s_M[head];
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const float4 r = make_float4(acc[i].x * inv, acc[i].y * inv, acc[i].z * inv, acc[i].w * inv);
    const float lse2 = L > 0.f ? M + __log2f(L) : -INFINITY;
    if (to_output) {
      const size_t row = row0 + head;
      if (a.out_bf16) {
        const uint32_t lo = pack_bf16(r.x, r.y), hi = pack_bf16(r.z, r.w);
        *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + row * kHeadDim + d) = make_uint2(lo, hi);
      } else {
        *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + row * kHeadDim + d) = r;
      }
      if (d == 0 && a.lse) a.lse[row] = lse2 * kLn2;
    } else {
      *reinterpret_cast<float4*>(a.part_o + ((size_t)dst * G + head) * kHeadDim + d) = r;
      if (d == 0) a.part_lse[(size_t)dst * G + head] = lse2;
    }
  }
}

// Byte offset of 16-B chunk cd (0..15) of token t in a staged slice: two
// 16-row x 128-B halves (d 0..63, d 64..127), 128-byte swizzle (chunk ^= row % 8).
__device__ __forceinline__ uint32_t slice_off(int t, int cd) {
  return (uint32_t)((cd >> 3) * kHalfBytes + t * 128 + (((cd & 7) ^ (t & 7)) << 4));
}

#ifndef L4_EARLY_RELEASE
#define L4_EARLY_RELEASE 1
#endif
// One page (16 tokens) of one (request, kv head): S^T = K Q^T, online softmax, O^T += V^T P^T.
// With L4_EARLY_RELEASE the V fragments are loaded right after the S product and the stage is
// released to the producer (proxy fence, arrive on `rel_bar`) before the softmax and the PV
// product, so a stage is held only while it is read and the next TMA into it goes out sooner.
__device__ __forceinline__ void consume_page(uint32_t sbase, int valid, const uint32_t (&qf)[8][2],
                                             float (&acc)[8][4], float (&mrow)[2], float (&lrow)[2],
                                             float scale_log2, int lane, uint32_t& cks_k, uint32_t& cks_v,
                                             uint32_t rel_bar) {
  using namespace dev;
#ifdef L4_NO_COMPUTE  // measurement-only: the data-movement skeleton (ring, scheduling) without the math
  __syncwarp();
  if (lane == 0) mbar_arrive(rel_bar);
  return;
#endif
  const int g = lane >> 2, c = lane & 3;
  const int mi = lane >> 3, r8 = lane & 7;

  // ---- S^T[16 tok x 8 heads] = K[16 x 128] * Q^T[128 x 8]
  float s[4] = {0.f, 0.f, 0.f, 0.f};
  {
    const int tok = r8 + ((mi & 1) << 3);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      uint32_t a0, a1, a2, a3;
      ldmatrix_x4(sbase + slice_off(tok, kk * 2 + (mi >> 1)), a0, a1, a2, a3);
      cks_k ^= a0 ^ a1 ^ a2 ^ a3;  // debug checksum (dead code unless L4_DEBUG_CKS)
      mma_bf16_16816(s, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
    }
  }
#if L4_EARLY_RELEASE
  uint32_t vf[8][4];
  {
    const int tok = r8 + ((mi >> 1) << 3);
    const uint32_t vbase = sbase + kSliceBytes;
    // masks for invalid tokens of a partial last page (V may hold NaN there)
    const uint32_t mlo = (((2 * c) < valid) ? 0x0000ffffu : 0u) | (((2 * c + 1) < valid) ? 0xffff0000u : 0u);
    const uint32_t mhi = (((2 * c + 8) < valid) ? 0x0000ffffu : 0u) | (((2 * c + 9) < valid) ? 0xffff0000u : 0u);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      ldmatrix_x4_trans(vbase + slice_off(tok, mt * 2 + (mi & 1)), vf[mt][0], vf[mt][1], vf[mt][2], vf[mt][3]);
      if (valid < kPage) {
        vf[mt][0] &= mlo;
        vf[mt][1] &= mlo;
        vf[mt][2] &= mhi;
        vf[mt][3] &= mhi;
      }
      cks_v ^= vf[mt][0] ^ vf[mt][1] ^ vf[mt][2] ^ vf[mt][3];
    }
  }
  fence_proxy_async_smem();  // this warp's reads of the stage before the producer's next TMA into it
  __syncwarp();
  if (lane == 0) mbar_arrive(rel_bar);
#endif
  // ---- mask (Z20: tokens >= kv_len are not attended) and online softmax in the exp2 domain
  const float NEG = -INFINITY;
  const float t0 = (g < valid) ? s[0] * scale_log2 : NEG;
  const float t1 = (g < valid) ? s[1] * scale_log2 : NEG;
  const float t2 = (g + 8 < valid) ? s[2] * scale_log2 : NEG;
  const float t3 = (g + 8 < valid) ? s[3] * scale_log2 : NEG;
  float mx0 = fmaxf(t0, t2), mx1 = fmaxf(t1, t3);
#pragma unroll
  for (int o = 4; o < 32; o <<= 1) {
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
  }
  const float mn0 = fmaxf(mrow[0], mx0), mn1 = fmaxf(mrow[1], mx1);
  const float mu0 = (mn0 == NEG) ? 0.f : mn0, mu1 = (mn1 == NEG) ? 0.f : mn1;
  const float al0 = ex2(mrow[0] - mu0), al1 = ex2(mrow[1] - mu1);
  mrow[0] = mn0;
  mrow[1] = mn1;
  const float p0 = ex2(t0 - mu0), p1 = ex2(t1 - mu1), p2 = ex2(t2 - mu0), p3 = ex2(t3 - mu1);
  lrow[0] = lrow[0] * al0 + (p0 + p2);
  lrow[1] = lrow[1] * al1 + (p1 + p3);
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    acc[mt][0] *= al0;
    acc[mt][1] *= al1;
    acc[mt][2] *= al0;
    acc[mt][3] *= al1;
  }
  // ---- P^T as B fragments: bf16 hi + lo (Z23), transposed with movmatrix
  const uint32_t h0 = pack_bf16(p0, p1), h1 = pack_bf16(p2, p3);
  const uint32_t l0 = pack_bf16(p0 - bf16_lo_f(h0), p1 - bf16_hi_f(h0));
  const uint32_t l1 = pack_bf16(p2 - bf16_lo_f(h1), p3 - bf16_hi_f(h1));
  const uint32_t bh0 = movmatrix_trans(h0), bh1 = movmatrix_trans(h1);
  const uint32_t bl0 = movmatrix_trans(l0), bl1 = movmatrix_trans(l1);
  // ---- O^T[128 d x 8 heads] += V^T[128 x 16 tok] * P^T[16 tok x 8 heads]
#if L4_EARLY_RELEASE
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    mma_bf16_16816(acc[mt], vf[mt][0], vf[mt][1], vf[mt][2], vf[mt][3], bh0, bh1);
    mma_bf16_16816(acc[mt], vf[mt][0], vf[mt][1], vf[mt][2], vf[mt][3], bl0, bl1);
  }
#else
  {
    const int tok = r8 + ((mi >> 1) << 3);
    const uint32_t vbase = sbase + kSliceBytes;
    // masks for invalid tokens of a partial last page (V may hold NaN there)
    const uint32_t mlo = (((2 * c) < valid) ? 0x0000ffffu : 0u) | (((2 * c + 1) < valid) ? 0xffff0000u : 0u);
    const uint32_t mhi = (((2 * c + 8) < valid) ? 0x0000ffffu : 0u) | (((2 * c + 9) < valid) ? 0xffff0000u : 0u);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      uint32_t a0, a1, a2, a3;
      ldmatrix_x4_trans(vbase + slice_off(tok, mt * 2 + (mi & 1)), a0, a1, a2, a3);
      if (valid < kPage) {
        a0 &= mlo;
        a1 &= mlo;
        a2 &= mhi;
        a3 &= mhi;
      }
      cks_v ^= a0 ^ a1 ^ a2 ^ a3;
      mma_bf16_16816(acc[mt], a0, a1, a2, a3, bh0, bh1);
      mma_bf16_16816(acc[mt], a0, a1, a2, a3, bl0, bl1);
    }
  }
  fence_proxy_async_smem();  // this warp's reads of the stage before the producer's next TMA into it
  __syncwarp();
  if (lane == 0) mbar_arrive(rel_bar);
#endif
}

__device__ __forceinline__ WorkItem load_item(const WorkItem* items, int i, int n) {
  WorkItem it;
  if (i < n) {
    const int4* p = reinterpret_cast<const int4*>(items + i);
    const int4 x = __ldg(p), y = __ldg(p + 1);
    it.b = x.x; it.h = x.y; it.pbeg = x.z; it.pend = x.w;
    it.last_valid = y.x; it.part_base = y.y; it.nsplit = y.z; it.split = y.w;
  } else {
    it.b = -1; it.h = 0; it.pbeg = 0; it.pend = 0; it.last_valid = 0; it.part_base = 0; it.nsplit = 1; it.split = 0;
  }
  return it;
}


template <int G, bool kFused>
__global__ void __launch_bounds__(kThreads, 2)
    decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, RunArgs a) {
  using namespace dev;
  using SL = SmemLayout<G>;
  constexpr int kStages = SL::stages_n;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw_u32 & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + SL::bars;
  const uint32_t bar_empty = bar_full + kStages * 8;
  const uint32_t bar_ifull = bar_empty + kStages * 8;
  const uint32_t bar_iempty = bar_ifull + kItemSlots * 8;
  SlotItem* s_items = reinterpret_cast<SlotItem*>(smem + SL::items);
  float* merge_o = reinterpret_cast<float*>(smem + SL::merge_o);
  float* merge_m = reinterpret_cast<float*>(smem + SL::merge_m);
  float* merge_l = reinterpret_cast<float*>(smem + SL::merge_l);
  volatile int* s_flag = reinterpret_cast<volatile int*>(smem + SL::flag);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) L4_MARK(0);
  volatile int* s_seq = reinterpret_cast<volatile int*>(smem + SL::seq);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) s_seq[i] = -1;
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar_full + i * 8, 1);
      mbar_init(bar_empty + i * 8, 1);
    }
    for (int i = 0; i < kItemSlots; ++i) {
      mbar_init(bar_ifull + i * 8, 1);
      mbar_init(bar_iempty + i * 8, kConsumerThreads);  // every consumer thread releases its reads
    }
    fence_mbar_init();
  }
  if (warp == kConsumerWarps && lane == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
#if L4_PREFETCH_INPUTS
    // L2 prefetch of the inputs the prologue reads first — this CTA's share of the page ids and
    // of q, and (CTA 0) kv_len / indptr — so the plan's loads, the first units' page-id loads and
    // Q copies hit L2.  A hint, safe before griddepcontrol.wait even in plain mode: L2 is the
    // point of coherence, so a write of the previous kernel supersedes a prefetched line.
    const int W0 = gridDim.x;
    auto pf_share = [&](const void* base, long long bytes) {
      if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || bytes < 16) return;
      const long long share = ((bytes + W0 - 1) / W0 + 15) & ~15ll;
      const long long off = share * blockIdx.x;
      const long long len = min(share, bytes - off) & ~15ll;
      if (len > 0) prefetch_l2_bulk(static_cast<const char*>(base) + off, (uint32_t)len);
    };
    pf_share(a.indices, a.n_indices * 4);
    pf_share(a.q, (long long)a.B * a.Hq * kHeadDim * 2);
    if (kFused && blockIdx.x == 0) {
      const long long b16 = ((long long)a.B * 4) & ~15ll;
      if (b16 > 0 && ((reinterpret_cast<uintptr_t>(a.kv_len) | reinterpret_cast<uintptr_t>(a.indptr)) & 15) == 0) {
        prefetch_l2_bulk(a.kv_len, (uint32_t)b16);
        prefetch_l2_bulk(a.indptr, (uint32_t)b16);
      }
    }
#endif
  }
  __syncthreads();
  // PDL: the next kernel in the stream may start its prologue as CTAs of this one retire; it
  // waits (griddepcontrol.wait) for this grid to complete before touching memory.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // PDL: everything above overlapped the previous kernel (the planner, or the previous step).
  // Early mode (fused only): the plan and the first item's loads read only the caller's inputs,
  // which the previous kernel must not be writing (L4_DECODE_EARLY_INPUTS); every access to the
  // workspace and every output write still comes after griddepcontrol.wait.
  // Early-plan mode (L4_DECODE_EARLY_PLAN, fused only): the plan reads kv_len / indptr before
  // the wait (the kernel before must not write them: true in a decode step's layer loop, where
  // the page table is uploaded once per step), q / K / V and the workspace only after it.
  const bool early = kFused && a.early == 1;
  const bool early_plan = kFused && a.early == 2;
  if (!early && !early_plan) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) L4_MARK(1);

  const int W = gridDim.x;
  int n_items, plan_C = 0, n_wide, q_pages = 0;
  int *p_len = nullptr, *p_ptr = nullptr, *p_rb = nullptr, *p_off = nullptr;
  if constexpr (kFused) {
    // a1 in every CTA: the plan lives in this CTA's shared memory (scratch in the merge area,
    // free until the first item finishes); no planner launch and no global work list.
    p_len = reinterpret_cast<int*>(smem + SL::total);
    p_ptr = p_len + a.B;
    p_rb = p_ptr + a.B;
    p_off = p_rb + a.B;
    int pmax;
    plan_core(a.kv_len, a.indptr, a.B, a.Hkv, W, a.forced_chunk, a.items_cap, p_len, p_ptr, p_rb, p_off,
              smem + SL::merge_o, &plan_C, &n_items, &pmax, SL::quads ? a.quad_bin : 0, &n_wide, &q_pages);
  } else {
    n_items = a.header->n_items;
    n_wide = SL::quads ? a.header->n_wide : n_items;
    q_pages = a.header->quad_pages;
  }
  if (early_plan) asm volatile("griddepcontrol.wait;" ::: "memory");
  // Scheduling units: items [0, n_wide) one per unit (CTA-wide); then the quad-eligible suffix
  // four items per unit (one per consumer warp), except its last kQuadTailPerCta x W items,
  // which run CTA-wide again so the end of the launch has the fine granularity of single
  // items.  Quads only when every CTA gets several (a small batch keeps 4 warps per item: one
  // warp alone streams a page at a fraction of a CTA's share of HBM bandwidth).
  const int q_rest = n_items - n_wide;
  int n_quads = (q_rest - min(q_rest, kQuadTailPerCta * W)) / kQuad;
  // A quad is the launch's granularity at the end, so quads need q_pages / kQuadPagesPerUnitCta
  // units per CTA, at least 1 and at most kQuadMinPerCta (q_pages = pages of the largest quad
  // item).  Measured (plain calls, units per CTA -> quads vs CTA-wide items): 13-page items at
  // 1.7 / 2.0 / 3.5 per CTA 37.7 vs 42.2 / 49.9 vs 51.7 / 72.3 vs 80.0 us (70B shape: 38.9 vs
  // 51.0 at 1.7 per CTA); 25-page items at 1.35 per CTA 63.0 vs 57.3 (worse), at 2.7 99.7 vs
  // 103.8; 50-page items at 1.1 per CTA 114 vs 86 (worse).  (Round 1's rule, min(4, pages / 4)
  // per CTA, predates the quad pacing and epilogue of late round 2.)
  if (kQuadPagesPerUnitCta * n_quads < min(kQuadMinPerCta * kQuadPagesPerUnitCta, max(kQuadPagesPerUnitCta, q_pages)) * W)
    n_quads = 0;
  const int n_units = n_items - (kQuad - 1) * n_quads;
  const int u_tail = n_wide + n_quads;  // first tail unit
  if (threadIdx.x == 0) L4_MARK(2);
  auto get_item = [&](int i) -> WorkItem {
    if constexpr (kFused)
      return item_from_plan(i, n_items, p_len, p_ptr, p_rb, p_off, a.B, a.Hkv);
    else
      return load_item(a.items, i, n_items);
  };
  auto unit_item = [&](int u) -> int {
    return u < n_wide ? u : (u < u_tail ? n_wide + kQuad * (u - n_wide) : u + (kQuad - 1) * n_quads);
  };
  auto is_quad = [&](int u) -> bool { return u >= n_wide && u < u_tail; };

  if (warp == kConsumerWarps) {
    // ============================== producer warp: items, Q and KV pages via TMA
#ifdef L4_TRACE
    L4_TRACE_ACC
#endif
    const uint64_t policy = policy_evict_first();
    bool exhausted = false;
    // Dynamic LPT scheduling: the first unit is blockIdx.x, later ones come from an atomic
    // ticket (W + ticket) drawn when the current unit's pages are issued, so idle CTAs take the
    // next-largest unit and no CTA holds work it has not started when the counter runs out
    // (round 1 held three tickets ahead: C3 ended over an 80 us spread of CTA finish times).
    // The atomic's round trip is covered by the kStages pages the ring still holds.  Every
    // drawn ticket is resolved before this CTA reports done: the last CTA to report resets
    // the scheduler for the next run.
    auto resolve = [&](int raw) -> int {
      const int t = __shfl_sync(0xffffffffu, raw, 0);
      if (t < 0 || exhausted) return n_units;
      if (W + t >= n_units) {
        exhausted = true;
        return n_units;
      }
      return W + t;
    };
    auto issue = [&]() -> int {
      int t = -1;
      if (lane == 0 && !exhausted) t = atomicAdd(&a.header->sched_next, 1);
      return t;
    };
    auto post_item = [&](uint32_t kk, const WorkItem& it, int idx) {  // lane 0: item + its Q rows
      const uint32_t slot = kk % kItemSlots;
      mbar_wait(bar_iempty + slot * 8, ((kk / kItemSlots) & 1) ^ 1);
      s_items[slot].it[0] = it;
      s_items[slot].idx = idx;
      s_items[slot].nsub = 0;
      const uint32_t qbytes = G * kHeadDim * 2;
      mbar_arrive_expect_tx(bar_ifull + slot * 8, qbytes);
      bulk_load(sbase + SL::qslots + slot * SL::qslot_bytes,
                a.q + ((size_t)it.b * a.Hq + (size_t)it.h * G) * kHeadDim, qbytes, bar_ifull + slot * 8);
    };
    uint32_t qseq = 0;
    auto issue_page = [&](int page, int h) {  // lane 0: one (page, kv head) K + V slice
      const uint32_t st = qseq % kStages;
#ifdef L4_TRACE
      const unsigned long long tw0 = trace_now();
#endif
      mbar_wait(bar_empty + st * 8, ((qseq / kStages) & 1) ^ 1);
#ifdef L4_TRACE
      trace_add(14, trace_now() - tw0);
#endif
      const uint32_t fb = bar_full + st * 8;
      mbar_arrive_expect_tx(fb, kStageBytes);
      if constexpr (kStages % kConsumerWarps != 0)
        st_release_cta(sbase + SL::seq + st * 4, (int)qseq);  // stage armed for page qseq
      const int row = (page * a.Hkv + h) * kPage;
      const uint32_t dst = sbase + SL::stages + st * kStageBytes;
      tma_load_3d(dst, &tmK, 0, row, 0, fb, policy);
      tma_load_3d(dst + kSliceBytes, &tmV, 0, row, 0, fb, policy);
#ifdef L4_TRACE
      if (qseq == 0) L4_MARK(3);
#endif
    };
    auto issue_null = [&]() {  // lane 0: a stage with no data (a quad's shorter item)
      const uint32_t st = qseq % kStages;
      mbar_wait(bar_empty + st * 8, ((qseq / kStages) & 1) ^ 1);
      if constexpr (kStages % kConsumerWarps != 0) st_release_cta(sbase + SL::seq + st * 4, (int)qseq);
      mbar_arrive(bar_full + st * 8);
    };
    // ---- units, prepared one ahead.  While a quad unit's pages go out, the ticket that names
    // the next unit is drawn (kDrawAhead ring positions before the unit's end) and resolved, and
    // the next unit's lookups (its item(s) from the plan, the first 32 page ids of each item:
    // global loads) are issued (kResolveAhead positions before the end), so neither the atomic's
    // nor the page ids' round trip sits between two short units, where the ring would drain (a
    // 16-page unit is ~5 us of a CTA's share of HBM): B = 1024 x 64 tokens 53.0 -> 50.0 us.  A CTA
    // holds at most one unstarted unit, and only during its current unit's last kDrawAhead
    // positions (round 1 held three tickets for whole units: an 80 us finish spread).  CTA-wide
    // units draw at their end (the ring's kStages pages cover the round trips there; a pacing
    // call in their page loop measured 1-2% slower on C2 / C4).
    struct Prep {
      WorkItem my;             // wide unit: the item (every lane); quad unit: item f + (lane & 3)
      int ids[kQuad][2];       // wide: ids[0][0] = page id `lane`; quad: ids j = lane, 32 + lane of item w
    };
    auto prep = [&](Prep& P, int u) {
      if (u >= n_units) return;
      if (SL::quads && is_quad(u)) {
        P.my = get_item(unit_item(u) + (lane & (kQuad - 1)));
#pragma unroll
        for (int w = 0; w < kQuad; ++w) {
          const int n = __shfl_sync(0xffffffffu, P.my.pend - P.my.pbeg, w);
          const int pb = __shfl_sync(0xffffffffu, P.my.pbeg, w);
          P.ids[w][0] = lane < n ? __ldg(a.indices + pb + lane) : 0;
          P.ids[w][1] = lane + 32 < n ? __ldg(a.indices + pb + 32 + lane) : 0;
        }
      } else {
        P.my = get_item(unit_item(u));
        P.ids[0][0] = lane < P.my.pend - P.my.pbeg ? __ldg(a.indices + P.my.pbeg + lane) : 0;
      }
    };
    // ring positions left in the unit when the ticket is drawn / resolved and the next unit
    // prepared (measured, B = 1024 x 64 tokens: G = 4 16 / 8 -> 50.2 us, 8 / 4 -> 50.7; G = 8
    // 16 / 8 -> 48.2 us, 8 / 4 -> 48.5)
    constexpr int kDrawAhead = 16;
    constexpr int kResolveAhead = 8;
    bool may_draw = !early;                  // early mode: no ticket before griddepcontrol.wait
    bool drawn = false, resolved = false;
    int t_raw = -1, since = 0, i_next = n_units;
    Prep cp, nx;
    auto pace = [&](int rem) {  // warp-uniform: called before issuing ring position `rem` from the end
      if (!may_draw) return;
      if (!drawn) {
        if (rem <= kDrawAhead) {
          t_raw = issue();  // the atomic's result is first used at the resolve below
          drawn = true;
          since = 0;
        }
      } else if (!resolved && ++since >= 2 && rem <= kResolveAhead) {
        i_next = resolve(t_raw);
        resolved = true;
        prep(nx, i_next);
      }
    };
    // Quad unit u (items f .. f + 3, one per consumer warp, prepared in P): lane 0 posts the slot
    // and issues the Q rows into it (G <= 4; at G = 8 the consumers load them); page j of item w
    // goes out as ring page qbase' + 4 j + w (null stages pad the shorter items), so warp w always
    // owns the ring positions = w (mod 4) of the unit.
    auto issue_quad = [&](int u, uint32_t kk, const Prep& P) {
      if constexpr (SL::quads) {
        const int f = unit_item(u);
        const int nsub = kQuad;  // quad units are always full (the remainder runs CTA-wide)
        int npw[kQuad], hw[kQuad];
        int maxnp = 0;
#pragma unroll
        for (int w = 0; w < kQuad; ++w) {
          npw[w] = __shfl_sync(0xffffffffu, P.my.pend - P.my.pbeg, w);
          hw[w] = __shfl_sync(0xffffffffu, P.my.h, w);
          maxnp = max(maxnp, npw[w]);
        }
        const uint32_t slot = kk % kItemSlots;
        // lane 0 writes the whole slot (it waited for it and arrives on its full barrier)
        int* fld = reinterpret_cast<int*>(&s_items[slot]);
        if (lane == 0) mbar_wait(bar_iempty + slot * 8, ((kk / kItemSlots) & 1) ^ 1);
#pragma unroll
        for (int w = 0; w < kQuad; ++w) {
          const int v0 = __shfl_sync(0xffffffffu, P.my.b, w), v1 = hw[w];
          const int v2 = __shfl_sync(0xffffffffu, P.my.pbeg, w), v3 = __shfl_sync(0xffffffffu, P.my.pend, w);
          const int v4 = __shfl_sync(0xffffffffu, P.my.last_valid, w);
          const int v5 = __shfl_sync(0xffffffffu, P.my.part_base, w);
          const int v6 = __shfl_sync(0xffffffffu, P.my.nsplit, w), v7 = __shfl_sync(0xffffffffu, P.my.split, w);
          if (lane == 0) {
            int* d = fld + w * 8;
            d[0] = v0; d[1] = v1; d[2] = v2; d[3] = v3; d[4] = v4; d[5] = v5; d[6] = v6; d[7] = v7;
          }
        }
        if (lane == 0) {
          s_items[slot].idx = f;
          s_items[slot].nsub = nsub;
          s_items[slot].maxnp = maxnp;
        }
        __syncwarp();
        const uint32_t qbytes = G * kHeadDim * 2;
        if constexpr (SL::q_global) {
          // slot published without data: the consumer warps load their items' Q rows themselves
          if (lane == 0) mbar_arrive(bar_ifull + slot * 8);
        } else {
          if (lane == 0) mbar_arrive_expect_tx(bar_ifull + slot * 8, nsub * qbytes);
          __syncwarp();
#pragma unroll
          for (int w = 0; w < kQuad; ++w) {  // lane 0 (the lane that waited for the slot) loads Q
            const int qb = __shfl_sync(0xffffffffu, P.my.b, w);
            if (lane == 0 && w < nsub)
              bulk_load(sbase + SL::qslots + slot * SL::qslot_bytes + w * qbytes,
                        a.q + ((size_t)qb * a.Hq + (size_t)hw[w] * G) * kHeadDim, qbytes, bar_ifull + slot * 8);
          }
        }
        for (int j = 0; j < maxnp; ++j) {
          pace(kQuad * (maxnp - j));
#pragma unroll
          for (int w = 0; w < kQuad; ++w) {
            const int page = __shfl_sync(0xffffffffu, j < 32 ? P.ids[w][0] : P.ids[w][1], j & 31);
            if (lane == 0) {
              if (j < npw[w])
                issue_page(page, hw[w]);
              else
                issue_null();
            }
            ++qseq;
          }
        }
      }
    };
    // CTA-wide unit u (one item, prepared in P): lane 0 posts the item slot and its Q rows, then
    // the item's pages go out one ring position each (page ids 32 at a time, one block ahead).
    auto issue_wide = [&](int u, uint32_t kk, const Prep& P) {
      const WorkItem& it = P.my;
      if (lane == 0) post_item(kk, it, unit_item(u));
      const int np = it.pend - it.pbeg;
      int blk = P.ids[0][0];
      for (int j0 = 0; j0 < np; j0 += 32) {
        const int nb = (j0 + 32 + lane < np) ? __ldg(a.indices + it.pbeg + j0 + 32 + lane) : 0;
        const int cnt = min(32, np - j0);
        for (int j = 0; j < cnt; ++j) {
          const int page = __shfl_sync(0xffffffffu, blk, j);
          if (lane == 0) issue_page(page, it.h);
#ifdef L4_DEBUG_CKS
          if (lane == 0 && unit_item(u) < 16384)
            atomicAdd(&g_cks[unit_item(u) * 4 + 3], (unsigned)page * (unsigned)(j0 + j + 1));
#endif
          ++qseq;
        }
        blk = nb;
      }
    };
    auto issue_unit = [&](int u, uint32_t kk, const Prep& P) {
      if (is_quad(u))
        issue_quad(u, kk, P);
      else
        issue_wide(u, kk, P);
    };
    // The first unit (blockIdx.x: no ticket needed) goes out before anything else; in early mode
    // all of it, before griddepcontrol.wait (it may run while the previous kernel finishes).
    int i_cur = blockIdx.x < n_units ? (int)blockIdx.x : n_units;  // unit indices from here on
    if (i_cur >= n_units) exhausted = true;
    prep(cp, i_cur);
    bool first_done = false;
    if (early && i_cur < n_units) {
      issue_unit(i_cur, 0, cp);
      first_done = true;
    }
    // from here on the scheduler state of the workspace is touched
    if (early) asm volatile("griddepcontrol.wait;" ::: "memory");
    may_draw = true;
    uint32_t k = 0;
    for (; i_cur < n_units; ++k) {
      if (!(k == 0 && first_done)) issue_unit(i_cur, k, cp);
      if (!drawn) t_raw = issue();
      if (!resolved) {
        i_next = resolve(t_raw);
        prep(nx, i_next);
      }
      drawn = resolved = false;
      i_cur = i_next;
      cp = nx;
    }
    // every ticket this CTA drew has been resolved: report done
    if (lane == 0) {
      const int done = atomicAdd(&a.header->sched_done, 1);
      if (done == W - 1) {  // every CTA stopped drawing: reset for the next run
        a.header->sched_next = 0;
        a.header->sched_done = 0;
      }
    }
#ifdef L4_TRACE
    if (lane == 0) L4_TRACE_FLUSH(14);
#endif
    // sentinel: tell the consumers there is no more work
    if (lane == 0) {
      const uint32_t slot = k % kItemSlots;
      mbar_wait(bar_iempty + slot * 8, ((k / kItemSlots) & 1) ^ 1);
      s_items[slot].it[0].b = -1;
      s_items[slot].nsub = 0;
      mbar_arrive(bar_ifull + slot * 8);
    }
    return;
  }

  // ============================== consumer warps
#ifdef L4_TRACE
  L4_TRACE_ACC
#endif
  const int g = lane >> 2, c = lane & 3;
  const int ct = threadIdx.x;  // 0..127
  // split bookkeeping for the deferred two-level combine (see the epilogue below)
  auto group_need = [&](const WorkItem& w) -> int {
    const int g0 = (w.split / kCombineGroup) * kCombineGroup;
    return min(kCombineGroup, w.nsplit - g0);
  };
  auto group_ctr = [&](const WorkItem& w) -> int* {
    if (w.nsplit > kCombineGroup) return a.gcount + w.part_base + (w.split / kCombineGroup) * kCombineGroup;
    return a.counters + (size_t)w.b * a.Hkv + w.h;
  };
  auto finish_group = [&](const WorkItem& w) {  // this CTA was the last split of w's group
    const int ns = w.nsplit;
    const int ng = (ns + kCombineGroup - 1) / kCombineGroup;
    const int g0 = (w.split / kCombineGroup) * kCombineGroup;
    const size_t row0 = (size_t)w.b * a.Hq + (size_t)w.h * G;
    combine_slots<G>(a, merge_o, w.part_base + g0, 1, group_need(w), ng == 1, row0, w.part_base + g0, ct);
    if (ng > 1) {
      named_bar_sync(1, kConsumerThreads);
      if (ct == 0) {
        int* ctr = a.counters + (size_t)w.b * a.Hkv + w.h;
        const int old = atom_add_acq_rel_gpu(ctr, 1);
        const int last = (old == ng - 1);
        if (last) *ctr = 0;
        *s_flag = last;
      }
      named_bar_sync(1, kConsumerThreads);
      if (*s_flag) combine_slots<G>(a, merge_o, w.part_base, kCombineGroup, ng, true, row0, 0, ct);
    }
  };
  bool has_pend = false;
  WorkItem pend_it;
  pend_it.b = -1;
  int pend_old = 0;
  uint32_t qbase = 0;
  for (uint32_t k = 0;; ++k) {
    const uint32_t slot = k % kItemSlots;
#ifdef L4_TRACE
    const unsigned long long ti0 = trace_now();
#endif
    mbar_wait(bar_ifull + slot * 8, (k / kItemSlots) & 1);
#ifdef L4_TRACE
    if (ct == 0) trace_add(10, trace_now() - ti0);
#endif
    const int nsub = s_items[slot].nsub;
    if (SL::quads && nsub > 0) {
      // ---- quad unit: this warp runs item `warp` alone (ring pages qbase + 4 j + warp) and
      // writes its output; no merge, no CTA barrier (warps drift freely across quad units)
      const int maxnp = s_items[slot].maxnp;
      const bool mine = warp < nsub;
      const WorkItem it = s_items[slot].it[mine ? warp : 0];
      uint32_t qf[8][2];
      auto load_qf = [&](const unsigned char* qs) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          if (g < G && mine) {
            qf[kk][0] = *reinterpret_cast<const uint32_t*>(qs + g * 256 + (kk * 16 + 2 * c) * 2);
            qf[kk][1] = *reinterpret_cast<const uint32_t*>(qs + g * 256 + (kk * 16 + 8 + 2 * c) * 2);
          } else {
            qf[kk][0] = 0u;
            qf[kk][1] = 0u;
          }
        }
      };
      if constexpr (SL::q_global) {
        // G = 8: the item's 8 Q rows straight from global memory into the mma B fragments (16
        // independent 4-byte loads per lane, in flight while the item's first page arrives), so
        // no ring position carries 2 KB of Q in an 8 KB stage
        mbar_arrive(bar_iempty + slot * 8);  // the slot was read above
        const __nv_bfloat16* qr = a.q + ((size_t)it.b * a.Hq + (size_t)it.h * G + g) * kHeadDim;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          qf[kk][0] = __ldg(reinterpret_cast<const unsigned*>(qr + kk * 16 + 2 * c));
          qf[kk][1] = __ldg(reinterpret_cast<const unsigned*>(qr + kk * 16 + 8 + 2 * c));
        }
      } else {
        load_qf(smem + SL::qslots + slot * SL::qslot_bytes + warp * (G * kHeadDim * 2));
        fence_proxy_async_smem();  // Q-slot reads before the producer's next bulk copy into the slot
        __syncwarp();
        mbar_arrive(bar_iempty + slot * 8);
      }
      float acc[8][4];
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
      float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
      uint32_t cks_k = 0, cks_v = 0;
      const int np = mine ? it.pend - it.pbeg : 0;
      for (int j = 0; j < maxnp; ++j) {
        const uint32_t q = qbase + kQuad * j + warp;
        const uint32_t st = q % kStages;
        if constexpr (kStages % kConsumerWarps != 0) {
          while (ld_acquire_cta(sbase + SL::seq + st * 4) != (int)q) {
          }
        }
        mbar_wait(bar_full + st * 8, (q / kStages) & 1);
        if (j < np) {  // consume_page releases the stage
          consume_page(sbase + SL::stages + st * kStageBytes, (j == np - 1) ? it.last_valid : kPage, qf, acc, mrow,
                       lrow, a.scale_log2, lane, cks_k, cks_v, bar_empty + st * 8);
        } else {  // a null stage (nothing was read)
          __syncwarp();
          if (lane == 0) mbar_arrive(bar_empty + st * 8);
        }
      }
      qbase += kQuad * maxnp;
      if (early && k == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // before any global write
      if (mine) {
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          lrow[0] += __shfl_xor_sync(0xffffffffu, lrow[0], o);
          lrow[1] += __shfl_xor_sync(0xffffffffu, lrow[1], o);
        }
        const size_t row0 = (size_t)it.b * a.Hq + (size_t)it.h * G;
        // Stage the item's G x 128 outputs in this warp's slice of the merge area (free in the
        // quad phase: the CTA-wide items that use it all precede the quads, behind CTA barriers),
        // then write each head row with one coalesced 16-byte-per-lane store: the fragment layout
        // scattered 32 four-byte stores per thread (with a division each), ~19% of the warp stall
        // samples of a B = 1024 x 64-token launch.
        float* so = merge_o + warp * (G * kMergeStride);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int head = 2 * c + hh;
          if (head < G) {
            const bool any = mrow[hh] != -INFINITY;
            const float inv = any ? 1.f / lrow[hh] : 0.f;
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
              so[head * kMergeStride + mt * 16 + g] = acc[mt][hh] * inv;
              so[head * kMergeStride + mt * 16 + g + 8] = acc[mt][2 + hh] * inv;
            }
            if (g == 0 && a.lse) a.lse[row0 + head] = any ? (mrow[hh] + __log2f(lrow[hh])) * kLn2 : -INFINITY;
          }
        }
        __syncwarp();
        if (a.out_bf16) {
#pragma unroll
          for (int head = 0; head < G; ++head) {
            const float4 r = *reinterpret_cast<const float4*>(so + head * kMergeStride + 4 * lane);
            *reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(a.out) + (row0 + head) * kHeadDim + 4 * lane) =
                make_uint2(pack_bf16(r.x, r.y), pack_bf16(r.z, r.w));
          }
        } else {
#pragma unroll
          for (int head = 0; head < G; ++head)
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(a.out) + (row0 + head) * kHeadDim + 4 * lane) =
                *reinterpret_cast<const float4*>(so + head * kMergeStride + 4 * lane);
        }
        __syncwarp();  // the slice is rewritten by this warp's next quad item
      }
      continue;
    }
    const WorkItem it = s_items[slot].it[0];
    const int item_idx = s_items[slot].idx;
    if (it.b < 0) break;
#ifdef L4_TRACE
    if (ct == 0) {
      g_trace_last[blockIdx.x * 4 + 0] = trace_now();
      g_trace_last[blockIdx.x * 4 + 1] = (unsigned long long)(it.pend - it.pbeg);
      g_trace_last[blockIdx.x * 4 + 2] = (unsigned long long)it.nsplit;
      g_trace_last[blockIdx.x * 4 + 3] = (unsigned long long)item_idx;
    }
#endif
    uint32_t qf[8][2];
    {
      const unsigned char* qs = smem + SL::qslots + slot * SL::qslot_bytes;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (g < G) {
          qf[kk][0] = *reinterpret_cast<const uint32_t*>(qs + g * 256 + (kk * 16 + 2 * c) * 2);
          qf[kk][1] = *reinterpret_cast<const uint32_t*>(qs + g * 256 + (kk * 16 + 8 + 2 * c) * 2);
        } else {
          qf[kk][0] = 0u;
          qf[kk][1] = 0u;
        }
      }
    }
    fence_proxy_async_smem();  // Q-slot reads before the producer's next bulk copy into the slot
    __syncwarp();
    mbar_arrive(bar_iempty + slot * 8);

    float acc[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    uint32_t cks_k = 0, cks_v = 0;
    const int np = it.pend - it.pbeg;
    for (int j = warp; j < np; j += kConsumerWarps) {
      const uint32_t q = qbase + j;
      const uint32_t st = q % kStages;
#ifdef L4_TRACE
      const unsigned long long tw0 = trace_now();
#endif
      if constexpr (kStages % kConsumerWarps != 0) {
        while (ld_acquire_cta(sbase + SL::seq + st * 4) != (int)q) {
        }
      }
      mbar_wait(bar_full + st * 8, (q / kStages) & 1);
#ifdef L4_TRACE
      if (q == 0 && lane == 0) L4_MARK(4);
      if (warp == 0 && lane == 0) trace_add(12, trace_now() - tw0);
#endif
      const int valid = (j == np - 1) ? it.last_valid : kPage;
#ifdef L4_TRACE
      const unsigned long long tc0 = trace_now();
#endif
      consume_page(sbase + SL::stages + st * kStageBytes, valid, qf, acc, mrow, lrow, a.scale_log2, lane, cks_k, cks_v,
                   bar_empty + st * 8);  // releases the stage
#ifdef L4_TRACE
      if (warp == 0 && lane == 0) trace_add(11, trace_now() - tc0);
#endif
    }
    qbase += np;
    if (early && k == 0) asm volatile("griddepcontrol.wait;" ::: "memory");  // before any global write
#ifdef L4_DEBUG_CKS
    {
      uint32_t cq = 0;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) cq ^= qf[kk][0] ^ (qf[kk][1] * 3u);
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        cks_k ^= __shfl_xor_sync(0xffffffffu, cks_k, o);
        cks_v ^= __shfl_xor_sync(0xffffffffu, cks_v, o);
        cq ^= __shfl_xor_sync(0xffffffffu, cq, o);
      }
      if (lane == 0 && item_idx < 16384) {
        atomicXor(&g_cks[item_idx * 4 + 0], cks_k * (2u * warp + 1u));
        atomicXor(&g_cks[item_idx * 4 + 1], cks_v * (2u * warp + 1u));
        if (warp == 0) atomicXor(&g_cks[item_idx * 4 + 2], cq);
      }
    }
#endif
#ifdef L4_TRACE
    const unsigned long long te0 = trace_now();
#endif

    // ---- intra-CTA merge of the 4 warps' (m, l, O)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      lrow[0] += __shfl_xor_sync(0xffffffffu, lrow[0], o);
      lrow[1] += __shfl_xor_sync(0xffffffffu, lrow[1], o);
    }
    {
      float* mo = merge_o + warp * (G * kMergeStride);
      const int h0 = 2 * c, h1 = 2 * c + 1;
      if (h0 < G) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          mo[h0 * kMergeStride + mt * 16 + g] = acc[mt][0];
          mo[h0 * kMergeStride + mt * 16 + g + 8] = acc[mt][2];
        }
        if (g == 0) {
          merge_m[warp * kMaxG + h0] = mrow[0];
          merge_l[warp * kMaxG + h0] = lrow[0];
        }
      }
      if (h1 < G) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          mo[h1 * kMergeStride + mt * 16 + g] = acc[mt][1];
          mo[h1 * kMergeStride + mt * 16 + g + 8] = acc[mt][3];
        }
        if (g == 0) {
          merge_m[warp * kMaxG + h1] = mrow[1];
          merge_l[warp * kMaxG + h1] = lrow[1];
        }
      }
    }
    named_bar_sync(1, kConsumerThreads);
    const bool split = it.nsplit > 1;
#pragma unroll
    for (int o = ct; o < G * kHeadDim; o += kConsumerThreads) {
      const int head = o / kHeadDim, d = o % kHeadDim;
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) M = fmaxf(M, merge_m[w * kMaxG + head]);
      float val = 0.f, lse2 = -INFINITY;
      if (M != -INFINITY) {
        float sum = 0.f, L = 0.f;
#pragma unroll
        for (int w = 0; w < kConsumerWarps; ++w) {
          const float sc = ex2(merge_m[w * kMaxG + head] - M);
          sum += sc * merge_o[w * (G * kMergeStride) + head * kMergeStride + d];
          L += sc * merge_l[w * kMaxG + head];
        }
        val = sum / L;
        lse2 = M + __log2f(L);
      }
      if (!split) {
        const size_t row = (size_t)it.b * a.Hq + (size_t)it.h * G + head;
        store_out(a, row * kHeadDim + d, val);
        if (d == 0 && a.lse) a.lse[row] = lse2 * kLn2;
      } else {
        const size_t prow = (size_t)item_idx * G + head;  // partial slot = item index
        a.part_o[prow * kHeadDim + d] = val;
        if (d == 0) a.part_lse[prow] = lse2;
      }
    }
    // ---- a3, two-level and deferred.  Split s belongs to group s / 16: the last split of a
    // group to finish combines the group's partials into the group's first slot, and the last
    // group of (b, kv head) to finish combines the group partials into the output; one combine
    // reads at most 32 partials (<= 512 splits).  The group ticket of a split item is issued
    // here but resolved at the end of this CTA's NEXT item, so no consumer waits for an atomic
    // round trip between items.  Counters are self-cleaning (reset by the last arrival).
    // Release: bar.sync orders every thread's partial stores before thread 0's acq_rel ticket
    // (cumulative); acquire: the ticket, then bar.sync, then ld.global.cg reads.  An unsplit item
    // with no pending ticket needs only the final barrier (merge area free).
    if (split || has_pend) named_bar_sync(1, kConsumerThreads);
    if (has_pend && ct == 0) {
      const int last = (pend_old == group_need(pend_it) - 1);
      if (last) *group_ctr(pend_it) = 0;
      *s_flag = last;
    }
    if (split && ct == 0) pend_old = atom_add_acq_rel_gpu(group_ctr(it), 1);
    if (has_pend) {
      named_bar_sync(1, kConsumerThreads);
      if (*s_flag) finish_group(pend_it);
    }
    has_pend = split;
    if (split) pend_it = it;
    named_bar_sync(1, kConsumerThreads);  // merge area free for the next item
#ifdef L4_TRACE
    if (ct == 0) {
      trace_add(13, trace_now() - te0);
      trace_add(15, 1);
    }
#endif
  }
  if (has_pend) {  // the last split item's ticket
    if (ct == 0) {
      const int last = (pend_old == group_need(pend_it) - 1);
      if (last) *group_ctr(pend_it) = 0;
      *s_flag = last;
    }
    named_bar_sync(1, kConsumerThreads);
    if (*s_flag) finish_group(pend_it);
  }
  if (threadIdx.x == 0) {
    L4_MARK(5);
#ifdef L4_TRACE
    L4_TRACE_FLUSH(10);
    L4_TRACE_FLUSH(11);
    L4_TRACE_FLUSH(12);
    L4_TRACE_FLUSH(13);
    L4_TRACE_FLUSH(15);
#endif
  }
}

// =================================================================== host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    cudaGetLastError();
  });
  return fn;
}

// Pool [num_pages, Hkv, 16, 128] bf16 viewed as a 3-D tensor
// (64 columns, num_pages*Hkv*16 rows of 256 B, 2 column halves 128 B apart);
// one box = 64 x 16 x 2 = one whole (page, kv head) slice of 4 KB, landing in
// shared memory as two 16-row x 128-B halves with the 128-byte swizzle.
l4_status make_tmap(CUtensorMap* tm, const void* base, int64_t rows) {
  auto enc = get_encode_fn();
  if (!enc) return fail(L4_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old or no device)");
  if (rows <= 0 || rows > ((int64_t)1 << 32)) return fail(L4_ERR_INVALID_ARG, "KV pool too large for a tensor map");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail(L4_ERR_INVALID_ARG, "KV pool must be 16-byte aligned");
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {(cuuint64_t)kHeadDim * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)kPage, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (CUresult %d)", (int)r);
    return L4_ERR_CUDA;
  }
  return L4_OK;
}

template <int G, bool kFused>
l4_status launch_decode(const CUtensorMap& tk, const CUtensorMap& tv, const RunArgs& a,
                        int grid, cudaStream_t st) {
  static std::atomic<bool> attr_set[64];  // per device; cudaFuncSetAttribute is idempotent
  const size_t smem_max = SmemLayout<G>::alloc + (kFused ? fused_plan_bytes(kFusedMaxBatch) : 0);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev].load(std::memory_order_acquire)) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<G, kFused>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem_max);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(decode_kernel<G, kFused>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      cudaGetLastError();
      return L4_ERR_CUDA;
    }
    attr_set[dev].store(true, std::memory_order_release);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SmemLayout<G>::alloc + (kFused ? fused_plan_bytes(a.B) : 0);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: overlap with the previous kernel
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, decode_kernel<G, kFused>, tk, tv, a);
  if (e != cudaSuccess) {
    set_error("decode_kernel launch failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  return L4_OK;
}

l4_status device_ctas(int* ctas_out) {
  static std::atomic<int> cache[64];  // per device (0 = not queried yet); racing first calls agree
  int dev = 0;
  l4_status s = get_device(&dev);
  if (s != L4_OK) return s;
  if (dev < 64) {
    const int c = cache[dev].load(std::memory_order_relaxed);
    if (c > 0) {
      *ctas_out = c;
      return L4_OK;
    }
  }
  int sms = 0;
  cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e != cudaSuccess) {
    set_error("cudaDeviceGetAttribute: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) {
    set_error("l4 requires an sm_100a (B200) device; device %d has compute capability %d.x", dev, major);
    return L4_ERR_CUDA;
  }
  const int ctas = sms * 2;  // two persistent CTAs per SM (~92 KB shared memory, 160 threads each)
  if (dev < 64) cache[dev].store(ctas, std::memory_order_relaxed);
  *ctas_out = ctas;
  return L4_OK;
}

}  // namespace
}  // namespace l4

using namespace l4;

extern "C" size_t l4_decode_workspace_size(const l4_decode_params* p, int64_t max_total_pages) {
  int G = 0;
  if (check_params(p, &G) != L4_OK) return 0;
  if (max_total_pages < 0) {
    set_error("max_total_pages < 0");
    return 0;
  }
  int ctas = 0;
  if (device_ctas(&ctas) != L4_OK) return 0;
  const int cap = items_cap_for(p, max_total_pages, ctas);
  return ws_layout(p->batch, p->num_kv_heads, G, cap).total;
}

#ifdef L4_DEBUG_CKS
extern "C" int l4_debug_cks(unsigned* host, int n, int clear) {
  if (clear) {
    void* p = nullptr;
    cudaGetSymbolAddress(&p, g_cks);
    return (int)cudaMemset(p, 0, sizeof(unsigned) * 16384 * 4);
  }
  return (int)cudaMemcpyFromSymbol(host, g_cks, sizeof(unsigned) * (size_t)n);
}
#endif
#ifdef L4_TRACE
extern "C" int l4_trace_read(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * (size_t)n);
}
extern "C" int l4_trace_read_last(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace_last, sizeof(unsigned long long) * (size_t)n);
}
extern "C" int l4_trace_clear(void) {
  static unsigned long long zeros[4096 * 16];
  return (int)cudaMemcpyToSymbol(g_trace, zeros, sizeof(zeros));
}
__device__ unsigned long long g_trace_stamp[64];
__global__ void trace_stamp_kernel(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_trace_stamp[slot] = t;
}
// stream-ordered globaltimer stamp (a 1-thread kernel): brackets a call on the GPU timeline
extern "C" int l4_trace_stamp(int slot, void* stream) {
  trace_stamp_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(slot);
  return (int)cudaGetLastError();
}
extern "C" int l4_trace_read_stamps(unsigned long long* host, int n) {
  return (int)cudaMemcpyFromSymbol(host, g_trace_stamp, sizeof(unsigned long long) * (size_t)n);
}
#endif

extern "C" l4_status l4_decode_workspace_init(const l4_decode_params* p, void* workspace, size_t workspace_bytes,
                                             void* stream) {
  int G = 0;
  l4_status s = check_params(p, &G);
  if (s != L4_OK) return s;
  if (!workspace) return fail(L4_ERR_WORKSPACE, "workspace is NULL");
  WsLayout L;
  if (!ws_layout_from_bytes(p->batch, p->num_kv_heads, G, workspace_bytes, &L))
    return fail(L4_ERR_WORKSPACE, "workspace too small");
  const size_t head = L.items;  // header + split counters + group counters
  cudaError_t e = cudaMemsetAsync(workspace, 0, head, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("cudaMemsetAsync: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  return L4_OK;
}

extern "C" l4_status l4_decode_workspace_regions(const l4_decode_params* p, size_t workspace_bytes,
                                                 l4_workspace_regions* out) {
  int G = 0;
  l4_status s = check_params(p, &G);
  if (s != L4_OK) return s;
  L4_CHECK_ARG(out != nullptr, "out is NULL");
  WsLayout L;
  if (!ws_layout_from_bytes(p->batch, p->num_kv_heads, G, workspace_bytes, &L))
    return fail(L4_ERR_WORKSPACE, "workspace too small");
  out->state_bytes = L.items;
  out->partial_lse_offset = L.part_lse;
  out->partial_o_offset = L.part_o;
  out->end_offset = L.part_o + (size_t)L.items_cap * G * kHeadDim * sizeof(float);
  out->items_cap = L.items_cap;
  out->group_size = G;
  return L4_OK;
}

static l4_status plan_impl(const l4_decode_params* p, const int32_t* kv_len, const int32_t* page_indptr,
                           int64_t total_pages, void* workspace, size_t workspace_bytes, cudaStream_t st) {
  int G = 0;
  l4_status s = check_params(p, &G);
  if (s != L4_OK) return s;
  L4_CHECK_ARG(total_pages >= 0, "total_pages < 0");
  if (p->batch > 0) L4_CHECK_ARG(kv_len && page_indptr, "kv_len / page_indptr is NULL");
  if (!workspace) return fail(L4_ERR_WORKSPACE, "workspace is NULL");
  int ctas = 0;
  s = device_ctas(&ctas);
  if (s != L4_OK) return s;
  const size_t need = ws_layout(p->batch, p->num_kv_heads, G, items_cap_for(p, total_pages, ctas)).total;
  WsLayout L;
  if (workspace_bytes < need || !ws_layout_from_bytes(p->batch, p->num_kv_heads, G, workspace_bytes, &L)) {
    set_error("workspace too small: %zu < %zu bytes (l4_decode_workspace_size)", workspace_bytes, need);
    return L4_ERR_WORKSPACE;
  }
  char* ws = static_cast<char*>(workspace);
  PlanArgs a;
  a.kv_len = kv_len;
  a.indptr = page_indptr;
  a.B = p->batch;
  a.Hkv = p->num_kv_heads;
  a.num_ctas = ctas;
  a.forced_chunk = p->chunk_pages;
  a.items_cap = L.items_cap;
  a.quad_bin = kQuadBin;
  a.header = reinterpret_cast<PlanHeader*>(ws + L.header);
  a.items = reinterpret_cast<WorkItem*>(ws + L.items);
  a.counters = reinterpret_cast<int*>(ws + L.counters);
  const size_t smem = kPlanScratchBytes + ((size_t)4 * std::max(p->batch, 1) + 1) * sizeof(int);
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kPlanScratchBytes + (4 * kMaxBatch + 1) * (int)sizeof(int));
    // same L1/shared carveout as decode_kernel: no SM reconfiguration between the two launches
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
  });
  // one warp per 32 requests (>= 4 warps, <= 32): latency, not throughput, bounds this kernel
  const int threads = std::min(kPlanThreads, std::max(128, (p->batch + 31) / 32 * 32));
  plan_kernel<<<1, threads, smem, st>>>(a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("plan_kernel launch failed: %s", cudaGetErrorString(e));
    return L4_ERR_CUDA;
  }
  return L4_OK;
}

// Shared by l4_decode_run (plan read from the workspace) and the fused l4_decode_attention
// (kv_len / page_indptr != NULL: every CTA plans in shared memory).
static l4_status run_impl(const l4_decode_params* p, const void* q, const void* k_pages, const void* v_pages,
                          int64_t num_pages, const int32_t* page_indices, void* out, float* lse, void* workspace,
                          size_t workspace_bytes, cudaStream_t st, const int32_t* kv_len = nullptr,
                          const int32_t* page_indptr = nullptr, int64_t total_pages = 0) {
  int G = 0;
  l4_status s = check_params(p, &G);
  if (s != L4_OK) return s;
  if (p->batch == 0) return L4_OK;
  const bool fused = kv_len != nullptr;
  // page_indices may be NULL only when every request is empty (indptr[B] == 0).
  L4_CHECK_ARG(q && k_pages && v_pages && out, "q/k_pages/v_pages/out is NULL");
  L4_CHECK_ARG(num_pages >= 1, "num_pages must be >= 1");
  L4_CHECK_ARG((reinterpret_cast<uintptr_t>(q) & 15) == 0, "q must be 16-byte aligned");
  if (!workspace) return fail(L4_ERR_WORKSPACE, "workspace is NULL");
  int ctas = 0;
  s = device_ctas(&ctas);
  if (s != L4_OK) return s;
  WsLayout L;
  if (fused) {
    L4_CHECK_ARG(page_indptr != nullptr, "page_indptr is NULL");
    L4_CHECK_ARG(total_pages >= 0, "total_pages < 0");
    const size_t need = ws_layout(p->batch, p->num_kv_heads, G, items_cap_for(p, total_pages, ctas)).total;
    if (workspace_bytes < need || !ws_layout_from_bytes(p->batch, p->num_kv_heads, G, workspace_bytes, &L)) {
      set_error("workspace too small: %zu < %zu bytes (l4_decode_workspace_size)", workspace_bytes, need);
      return L4_ERR_WORKSPACE;
    }
  } else if (!ws_layout_from_bytes(p->batch, p->num_kv_heads, G, workspace_bytes, &L)) {
    return fail(L4_ERR_WORKSPACE, "workspace too small");
  }
  const int64_t rows = num_pages * p->num_kv_heads * kPage;
  CUtensorMap tk, tv;
  s = make_tmap(&tk, k_pages, rows);
  if (s != L4_OK) return s;
  s = make_tmap(&tv, v_pages, rows);
  if (s != L4_OK) return s;
  char* ws = static_cast<char*>(workspace);
  RunArgs a;
  memset(&a, 0, sizeof(a));
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.out = out;
  a.lse = lse;
  a.indices = page_indices;
  a.items = reinterpret_cast<const WorkItem*>(ws + L.items);
  a.header = reinterpret_cast<PlanHeader*>(ws + L.header);
  a.counters = reinterpret_cast<int*>(ws + L.counters);
  a.gcount = reinterpret_cast<int*>(ws + L.gcount);
  a.part_o = reinterpret_cast<float*>(ws + L.part_o);
  a.part_lse = reinterpret_cast<float*>(ws + L.part_lse);
  a.Hq = p->num_q_heads;
  a.Hkv = p->num_kv_heads;
  const float scale = p->sm_scale > 0.f ? p->sm_scale : 1.0f / std::sqrt((float)kHeadDim);
  a.scale_log2 = scale * kLog2e;
  a.out_bf16 = p->out_dtype == L4_DT_BF16;
  a.kv_len = kv_len;
  a.indptr = page_indptr;
  a.B = p->batch;
  a.forced_chunk = p->chunk_pages;
  a.items_cap = L.items_cap;
  a.quad_bin = kQuadBin;
  a.early = !fused ? 0 : (p->flags & L4_DECODE_EARLY_INPUTS) ? 1 : (p->flags & L4_DECODE_EARLY_PLAN) ? 2 : 0;
  a.n_indices = fused ? total_pages : 0;
  if (fused) {
    switch (G) {
      case 1: return launch_decode<1, true>(tk, tv, a, ctas, st);
      case 2: return launch_decode<2, true>(tk, tv, a, ctas, st);
      case 4: return launch_decode<4, true>(tk, tv, a, ctas, st);
      default: return launch_decode<8, true>(tk, tv, a, ctas, st);
    }
  }
  switch (G) {
    case 1: return launch_decode<1, false>(tk, tv, a, ctas, st);
    case 2: return launch_decode<2, false>(tk, tv, a, ctas, st);
    case 4: return launch_decode<4, false>(tk, tv, a, ctas, st);
    default: return launch_decode<8, false>(tk, tv, a, ctas, st);
  }
}

extern "C" l4_status l4_decode_plan(const l4_decode_params* p, const int32_t* kv_len, const int32_t* page_indptr,
                                    int64_t total_pages, void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx("l4_decode_plan");
  if (p && p->batch == 0) {
    int G = 0;
    return check_params(p, &G);
  }
  return plan_impl(p, kv_len, page_indptr, total_pages, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" l4_status l4_decode_run(const l4_decode_params* p, const void* q, const void* k_pages, const void* v_pages,
                                   int64_t num_pages, const int32_t* page_indices, void* out, float* lse,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  NvtxRange nvtx("l4_decode_run");
  return run_impl(p, q, k_pages, v_pages, num_pages, page_indices, out, lse, workspace, workspace_bytes,
                  static_cast<cudaStream_t>(stream));
}

extern "C" l4_status l4_decode_attention(const l4_decode_params* p, const void* q, const void* k_pages,
                                         const void* v_pages, int64_t num_pages, const int32_t* page_indptr,
                                         const int32_t* page_indices, int64_t total_pages, const int32_t* kv_len,
                                         void* out, float* lse, void* workspace, size_t workspace_bytes,
                                         void* stream) {
  NvtxRange nvtx("l4_decode_attention");
  // One launch: every CTA of the decode kernel plans in its own shared memory (B <= 1024).
  // Larger batches: the materialised plan (planner kernel) followed by the run.
  int G = 0;
  const l4_status ps = check_params(p, &G);  // parameter errors first, as in plan / run
  if (ps != L4_OK) return ps;
  if (p->batch > 0 && p->batch <= kFusedMaxBatch) {
    L4_CHECK_ARG(kv_len != nullptr, "kv_len is NULL");
    return run_impl(p, q, k_pages, v_pages, num_pages, page_indices, out, lse, workspace, workspace_bytes,
                    static_cast<cudaStream_t>(stream), kv_len, page_indptr, total_pages);
  }
  l4_status s = l4_decode_plan(p, kv_len, page_indptr, total_pages, workspace, workspace_bytes, stream);
  if (s != L4_OK) return s;
  return l4_decode_run(p, q, k_pages, v_pages, num_pages, page_indices, out, lse, workspace, workspace_bytes, stream);
}

extern "C" l4_status l4_decode_plan_info(const void* workspace, l4_plan_info* info_out, void* stream) {
  L4_CHECK_ARG(workspace && info_out, "workspace / info_out is NULL");
  PlanHeader h;
  cudaError_t e = cudaMemcpyAsync(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) {
    set_error("plan_info copy failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  info_out->num_items = h.n_items;
  info_out->chunk_pages = h.chunk;
  info_out->num_ctas = h.num_ctas;
  info_out->max_splits = h.max_splits;
  info_out->tail_requests = h.tail_requests;
  info_out->tail_chunk_pages = h.tail_chunk;
  return L4_OK;
}

namespace l4 {
namespace {
// l4_decode_validate: one warp per request; report[0] counts violations, report[1..2] keep the
// lowest offending request and its kind (atomicMin on (request << 3 | kind)).
__global__ void validate_kernel(const int* kv_len, const int* indptr, const int* indices, int B, long long total_pages,
                                long long num_pages, int* owner, int* report) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= B) return;
  const int b = warp;
  const int L = kv_len[b];
  int kind = 0;
  long long np = 0, base = indptr[b];
  if (L < 0) {
    kind = 1;
  } else {
    np = (L + kPage - 1) / kPage;
    if (base < 0 || base + np > total_pages) kind = 2;
  }
  if (kind == 0) {
    for (long long j = lane; j < np; j += 32) {
      const int pg = indices[base + j];
      int k2 = 0;
      if (pg < 0 || pg >= num_pages) {
        k2 = 3;
      } else if (atomicCAS(owner + pg, -1, b) != -1) {
        k2 = 4;  // already claimed (by another request, or twice by this one)
      }
      const unsigned bad = __ballot_sync(__activemask(), k2 != 0);
      if (bad && kind == 0) kind = __shfl_sync(__activemask(), k2, __ffs(bad) - 1);
    }
    kind = __reduce_max_sync(0xffffffffu, kind);
  }
  if (lane == 0 && kind != 0) {
    atomicAdd(report, 1);
    atomicMin(report + 1, (b << 3) | kind);
  }
}
}  // namespace
}  // namespace l4

extern "C" l4_status l4_decode_validate(const l4_decode_params* p, const int32_t* kv_len, const int32_t* page_indptr,
                                        const int32_t* page_indices, int64_t total_pages, int64_t num_pages,
                                        int32_t* scratch, int32_t* report, void* stream) {
  int G = 0;
  l4_status s = check_params(p, &G);
  if (s != L4_OK) return s;
  L4_CHECK_ARG(report != nullptr, "report is NULL");
  L4_CHECK_ARG(total_pages >= 0 && num_pages >= 1, "total_pages < 0 or num_pages < 1");
  report[0] = 0;
  report[1] = -1;
  report[2] = 0;
  if (p->batch == 0) return L4_OK;
  L4_CHECK_ARG(kv_len && page_indptr && scratch, "kv_len / page_indptr / scratch is NULL");
  L4_CHECK_ARG(total_pages == 0 || page_indices, "page_indices is NULL");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* d_report = scratch + num_pages;  // [count, min(request << 3 | kind)] after the owner table
  static const int init[2] = {0, INT_MAX};
  cudaError_t e = cudaMemcpyAsync(d_report, init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(scratch, 0xff, (size_t)num_pages * sizeof(int), st);
  if (e == cudaSuccess) {
    const int threads = 256, blocks = (int)((p->batch * 32LL + threads - 1) / threads);
    validate_kernel<<<blocks, threads, 0, st>>>(kv_len, page_indptr, page_indices, p->batch, total_pages, num_pages,
                                                scratch, d_report);
    e = cudaGetLastError();
  }
  int h[2] = {0, INT_MAX};
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, d_report, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    set_error("l4_decode_validate: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  report[0] = h[0];
  report[1] = h[0] ? (h[1] >> 3) : -1;
  report[2] = h[0] ? (h[1] & 7) : 0;
  return L4_OK;
}

extern "C" l4_status l4_decode_plan_items(const void* workspace, int32_t* items_out, int32_t max_items, void* stream) {
  L4_CHECK_ARG(workspace && items_out && max_items >= 0, "bad arguments");
  PlanHeader h;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    const size_t gcount_off = align256(256 + (size_t)kMaxBatch * h.num_kv_heads * sizeof(int));
    const size_t items_off = align256(gcount_off + (size_t)h.items_cap * sizeof(int));
    const int n = std::min(h.n_items, max_items);
    if (n > 0)
      e = cudaMemcpyAsync(items_out, static_cast<const char*>(workspace) + items_off, (size_t)n * sizeof(WorkItem),
                          cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  if (e != cudaSuccess) {
    set_error("plan_items copy failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  return L4_OK;
}
