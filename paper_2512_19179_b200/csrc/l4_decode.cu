// l4_decode: length-binned split-KV GQA decode attention over a paged KV cache,
// for B200 (sm_100a).  Entry points: l4_decode_workspace_size / _plan / _run /
// _attention in include/l4.h.
//
// What is computed (definition in oracle/attention.py): for
// every request b and q-head h, softmax(scale * q K^T) V over the L_b cached
// tokens of kv head h/G, plus the natural-log LSE.
//
// How (B200 design):
//  a1  plan_kernel (1 CTA): pages -> chunk size C -> near-equal splits of the
//      requests longer than 2C -> work items binned by split length, longest
//      bin first (LPT order), so the longest request's splits start first and
//      short requests fill the tail (the paper's inter-SM imbalance and
//      partitioning inefficiency).  Zeroes the split counters and
//      the dynamic scheduler.
//  a2  decode_kernel (persistent, 1 producer + 4 consumer warps per CTA,
//      2 CTAs per SM): items are handed out dynamically (first one static,
//      then an atomic ticket), so CTAs that finish early take the next-largest
//      item.  The producer warp streams each (page, kv head) K and V slice
//      (4 KB each, HND layout) with one TMA each (cp.async.bulk.tensor, 128B
//      swizzle, L2 evict-first) into an 8-stage shared-memory ring tracked by
//      mbarriers; consumer warps compute S^T = K Q^T and O^T += V^T P^T with
//      mma.sync m16n8k16 (tokens / head_dim on M, the G <= 8 query heads on N,
//      so GQA group 8 has no padding), an online softmax with warp-shuffle max
//      reductions in the exp2 domain, and P split into bf16 hi + lo (Z23).
//  a3  LSE combine: the 4 warps of a CTA merge their (m, l, O) in shared
//      memory; a split item writes (O/l, lse) to the workspace and the last
//      split of (b, kv head) to finish (acq_rel atomic ticket) combines all
//      splits (FlashDecoding aggregation) — no second launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
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
constexpr int kStages = 8;
constexpr int kSliceBytes = kPage * kHeadDim * 2;     // one (page, kv head) K or V slice = 4 KB
constexpr int kHalfBytes = kSliceBytes / 2;           // 16 rows x 64 bf16 (128 B swizzle span)
constexpr int kStageBytes = 2 * kSliceBytes;          // K, V
constexpr int kItemSlots = 4;
constexpr int kMaxG = 8;
constexpr int kQSlotBytes = kMaxG * kHeadDim * 2;     // 2 KB
constexpr int kMergeStride = kHeadDim + 4;            // floats per head row (bank-conflict padding)
constexpr int kMaxSplits = 512;                       // per (request, kv head); lse staging capacity
constexpr int kMinChunk = 8;                          // pages
#ifndef L4_ITEMS_PER_CTA
#define L4_ITEMS_PER_CTA 8
#endif
constexpr int kItemsPerCta = L4_ITEMS_PER_CTA;        // automatic chunk target
constexpr int kNoSplitFactor = 2;                     // requests of <= 2C pages are never split
// Guided tail (planner): split the last requests of the LPT order into chunks of ~per-CTA/16.
// Measured r1: with the synchronous split epilogue it costs more than it saves (C2 151 -> 164 us),
// so it is disabled (kTailChunksPerCta = 0) until the epilogue is asynchronous.
constexpr int kTailChunksPerCta = 0;
constexpr int kTailDiv = 16;
constexpr int kMinTailChunk = 4;                      // pages
constexpr int kMaxBatch = 8192;
constexpr int kPlanThreads = 1024;
constexpr int kNumBins = 32;
constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;

struct __align__(16) WorkItem {
  int b, h, pbeg, pend, last_valid, part_base, nsplit, split;
};
static_assert(sizeof(WorkItem) == 32, "WorkItem is 32 bytes");

// Header region (256 B): plan summary + dynamic scheduler state.
struct __align__(16) PlanHeader {
  int n_items, chunk, num_ctas, max_splits;
  int batch, num_kv_heads, items_cap, pad;
  int tail_requests, tail_chunk, pad2[6];
  int sched_next, sched_done, pad3[14];  // ticket counter and finished-CTA count (self-resetting)
};
static_assert(sizeof(PlanHeader) == 128, "PlanHeader is 128 bytes");

// ------------------------------------------------------------------ workspace layout
struct WsLayout {
  size_t header, items, counters, part_lse, part_o, total;
  int items_cap;
};

inline size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

WsLayout ws_layout(int B, int Hkv, int G, int items_cap) {
  WsLayout L;
  L.items_cap = items_cap;
  L.header = 0;
  L.counters = 256;
  L.items = align256(L.counters + (size_t)std::max(B, 1) * Hkv * sizeof(int));
  L.part_lse = align256(L.items + (size_t)items_cap * sizeof(WorkItem));
  L.part_o = align256(L.part_lse + (size_t)items_cap * G * sizeof(float));
  L.total = align256(L.part_o + (size_t)items_cap * G * kHeadDim * sizeof(float));
  return L;
}

// The layout is a pure function of (B, Hkv, G, workspace_bytes): plan and run
// both derive the largest item capacity that fits the caller's workspace.
bool ws_layout_from_bytes(int B, int Hkv, int G, size_t bytes, WsLayout* out) {
  const WsLayout z = ws_layout(B, Hkv, G, 0);
  if (bytes < z.total) return false;
  const size_t per_item = sizeof(WorkItem) + (size_t)G * sizeof(float) + (size_t)G * kHeadDim * sizeof(float);
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
    // C >= T*Hkv/(W*k) => Hkv * sum ceil(p_b / C) <= W*k + Hkv*B
    cap = std::min(Hkv * (B + ceil_div64(max_total_pages, kMinChunk)),
                   Hkv * B + (int64_t)num_ctas * kItemsPerCta + Hkv) +
          (int64_t)num_ctas * kTailChunksPerCta + (kTailChunksPerCta > 0 ? Hkv * B : 0);  // guided-tail splits
  }
  cap = std::max<int64_t>(cap, 1);
  return (int)std::min<int64_t>(cap, INT_MAX / 64);
}

// =================================================================== a1: planner
struct PlanArgs {
  const int* kv_len;
  const int* indptr;
  int B, Hkv, num_ctas, forced_chunk, items_cap;
  PlanHeader* header;
  WorkItem* items;
  int* counters;
};

constexpr int kPlanMaxWarps = kPlanThreads / 32;

// Block-wide exclusive scan of one int per thread; returns the prefix, writes the total.
__device__ int block_excl_scan(int v, int* total, int* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  __syncthreads();
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int nw = blockDim.x >> 5;
    const int w = lane < nw ? s_warp[lane] : 0;
    int wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < nw) s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  *total = s_warp[32];
  return s_warp[warp] + incl - v;
}

// Block-wide (sum int64, max int, or bits) in one pass.
__device__ void block_reduce3(long long v, int m, unsigned bits, long long* s_ll, int* s_i, unsigned* s_u,
                              long long* sum_out, int* max_out, unsigned* or_out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    bits |= __shfl_xor_sync(0xffffffffu, bits, o);
  }
  __syncthreads();
  if (lane == 0) {
    s_ll[warp] = v;
    s_i[warp] = m;
    s_u[warp] = bits;
  }
  __syncthreads();
  long long t = 0;
  int mm = 0;
  unsigned bb = 0;
#pragma unroll 8
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
    t += s_ll[i];
    mm = max(mm, s_i[i]);
    bb |= s_u[i];
  }
  *sum_out = t;
  *max_out = mm;
  *or_out = bb;
}

__device__ __forceinline__ int pages_of(int L) { return L > 0 ? (L + kPage - 1) / kPage : 0; }

__device__ __forceinline__ int nsplit_of(int pages, int C) {
  if (pages <= kNoSplitFactor * C) return 1;  // also pages == 0
  return (pages + C - 1) / C;
}

__device__ __forceinline__ int bin_of(int pages, int nsplit) {
  if (pages <= 0) return 0;
  const int ip = (pages + nsplit - 1) / nsplit;  // pages of the largest split
  return min(kNumBins - 1, 32 - __clz(ip));      // bit_length(ip)
}

// One CTA of 1024 threads.  Requests are ordered by length bin, longest bin
// first, and by request index inside a bin (deterministic plans); each request
// contributes nsplit * Hkv items, contiguous per (request, kv head).
__global__ void __launch_bounds__(kPlanThreads, 1) plan_kernel(PlanArgs a) {
  // PDL: let the dependent decode kernel start its prologue now; it waits
  // (griddepcontrol.wait) for this grid's completion before reading the plan.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ int plan_smem[];  // s_len, s_ptr, s_rb (request at rank), s_off, s_ns (splits at rank)
  const int Bs = max(a.B, 1);
  int* s_len = plan_smem;
  int* s_ptr = plan_smem + Bs;
  int* s_rb = plan_smem + 2 * Bs;
  int* s_off = plan_smem + 3 * Bs;
  int* s_ns = plan_smem + 4 * Bs;
  __shared__ long long s_ll[32];
  __shared__ int s_i[33];
  __shared__ unsigned s_u[32];
  __shared__ int s_hist[kNumBins];
  __shared__ int s_binbase[kNumBins];
  __shared__ int s_wb[kPlanMaxWarps][kNumBins];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nthr = blockDim.x, nwarps = nthr >> 5;
  for (int b = tid; b < a.B; b += nthr) {
    s_len[b] = a.kv_len[b];
    s_ptr[b] = a.indptr[b];
  }
  if (tid < kNumBins) s_hist[tid] = 0;
  __syncthreads();

  long long T;
  int Pmax;
  unsigned unused;
  {
    long long sum = 0;
    int mx = 0;
    for (int b = tid; b < a.B; b += nthr) {
      const int pg = pages_of(s_len[b]);
      sum += pg;
      mx = max(mx, pg);
    }
    block_reduce3(sum, mx, 0u, s_ll, s_i, s_u, &T, &Pmax, &unused);
  }
  // chunk size C (pages per work item)
  long long Cl;
  if (a.forced_chunk > 0) {
    Cl = a.forced_chunk;
  } else if (a.forced_chunk < 0) {
    Cl = INT_MAX / 4;
  } else {
    const long long denom = (long long)a.num_ctas * kItemsPerCta;
    Cl = max((long long)kMinChunk, (T * a.Hkv + denom - 1) / denom);
  }
  Cl = max(Cl, (long long)((Pmax + kMaxSplits - 1) / kMaxSplits));
  int C = (int)min(Cl, (long long)(INT_MAX / 4));
  long long N;
  for (;;) {  // grow C until the work list fits the workspace (block-uniform loop)
    long long items = 0;
    for (int b = tid; b < a.B; b += nthr) items += (long long)nsplit_of(pages_of(s_len[b]), C) * a.Hkv;
    int dummy;
    block_reduce3(items, 0, 0u, s_ll, s_i, s_u, &N, &dummy, &unused);
    if (N <= a.items_cap || C >= INT_MAX / 8) break;
    C *= 2;
  }

  // ---- ranks: requests per bin, bins in descending order
  for (int t0 = 0; t0 < a.B; t0 += nthr) {  // warp-aggregated histogram of bins
    const int b = t0 + tid;
    int bin = -1;
    if (b < a.B) {
      const int pg = pages_of(s_len[b]);
      bin = bin_of(pg, nsplit_of(pg, C));
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && (peers & ((1u << lane) - 1u)) == 0) atomicAdd(&s_hist[bin], __popc(peers));
  }
  __syncthreads();
  if (warp == 0) {  // exclusive scan over bins, highest bin first
    const int bin = kNumBins - 1 - lane;
    const int h = s_hist[bin];
    int incl = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    s_binbase[bin] = incl - h;
  }
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int tile = 0; tile < a.B; tile += nthr) {  // block-uniform
    const int b = tile + tid;
    int bin = -1;
    if (b < a.B) {
      const int pg = pages_of(s_len[b]);
      bin = bin_of(pg, nsplit_of(pg, C));
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    const int lower = __popc(peers & lt_mask);
    __syncthreads();  // previous tile finished with s_wb / s_binbase
    for (int x = tid; x < nwarps * kNumBins; x += nthr) (&s_wb[0][0])[x] = 0;
    __syncthreads();
    if (bin >= 0 && lower == 0) s_wb[warp][bin] = __popc(peers);
    __syncthreads();
    if (tid < kNumBins) {  // per bin: exclusive running count over warps (request order)
      int run = 0;
      for (int w = 0; w < nwarps; ++w) {
        const int c = s_wb[w][tid];
        s_wb[w][tid] = run;
        run += c;
      }
      s_i[tid] = run;  // this tile's requests in bin tid
    }
    __syncthreads();
    if (bin >= 0) s_rb[s_binbase[bin] + s_wb[warp][bin] + lower] = b;
    __syncthreads();
    if (tid < kNumBins) s_binbase[tid] += s_i[tid];
  }
  __syncthreads();
  // ---- guided tail: the requests processed last (the suffix of the LPT order holding about
  // kTailChunksPerCta chunks of C_tail pages per CTA) are split into C_tail-page chunks so that
  // all CTAs finish within a small item of each other (auto mode only).
  const bool auto_mode = a.forced_chunk == 0;
  const long long per_cta = (T * a.Hkv + a.num_ctas - 1) / max(a.num_ctas, 1);
  const int Ct = (int)max((long long)kMinTailChunk, min((long long)C, (per_cta + kTailDiv - 1) / kTailDiv));
  const long long tail_budget = auto_mode ? (long long)kTailChunksPerCta * a.num_ctas * Ct : 0;
  int tail_requests = 0;
  if (kTailChunksPerCta == 0) {  // guided tail compiled out: plain splits
    for (int r = tid; r < a.B; r += nthr) s_ns[r] = nsplit_of(pages_of(s_len[s_rb[r]]), C);
  } else {
    long long carry = 0, extra = 0;
    int ntail = 0;
    for (int tile = 0; tile < a.B; tile += nthr) {  // exclusive prefix of page-heads in rank order
      const int r = tile + tid;
      const int pg = r < a.B ? pages_of(s_len[s_rb[r]]) : 0;
      int tot;
      const int ex = block_excl_scan(pg, &tot, s_i);
      if (r < a.B) {
        const long long suffix = (T - (carry + ex)) * a.Hkv;  // page-heads from rank r to the end
        int ns = nsplit_of(pg, C);
        if (suffix <= tail_budget && pg > 0) {
          const int nt = min(nsplit_of(pg, Ct), kMaxSplits);
          if (nt > ns) {
            extra += (long long)(nt - ns) * a.Hkv;
            ns = nt;
          }
          ntail += 1;
        }
        s_ns[r] = ns;
      }
      carry += tot;
    }
    long long ex_tot;
    int ntail_tot;
    unsigned unused2;
    block_reduce3(extra, ntail, 0u, s_ll, s_i, s_u, &ex_tot, &ntail_tot, &unused2);
    // block_reduce3's max is not a sum: count tail requests with a second pass
    int cnt = 0;
    for (int r = tid; r < a.B; r += nthr) cnt += s_ns[r] != nsplit_of(pages_of(s_len[s_rb[r]]), C) ? 1 : 0;
    long long cnt_ll;
    int dummy2;
    block_reduce3(cnt, 0, 0u, s_ll, s_i, s_u, &cnt_ll, &dummy2, &unused2);
    if (N + ex_tot > a.items_cap) {  // no room: keep the plain plan
      for (int r = tid; r < a.B; r += nthr) s_ns[r] = nsplit_of(pages_of(s_len[s_rb[r]]), C);
      ex_tot = 0;
      cnt_ll = 0;
    }
    N += ex_tot;
    tail_requests = (int)cnt_ll;
  }
  __syncthreads();
  // ---- item offsets: exclusive scan of nsplit * Hkv in rank order
  {
    int carry = 0;
    for (int tile = 0; tile < a.B; tile += nthr) {
      const int r = tile + tid;
      int cnt = 0;
      if (r < a.B) cnt = s_ns[r] * a.Hkv;
      int tot;
      const int ex = block_excl_scan(cnt, &tot, s_i);
      if (r < a.B) s_off[r] = carry + ex;
      carry += tot;
    }
  }
  __syncthreads();
  // ---- items: one thread per (request rank, kv head) writes that pair's splits
  for (int x = tid; x < a.B * a.Hkv; x += nthr) {
    const int r = x / a.Hkv, h = x - r * a.Hkv;
    const int b = s_rb[r];
    const int L = s_len[b];
    const int pg = pages_of(L);
    const int ns = s_ns[r];
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
    hd.n_items = (int)N;
    hd.chunk = C;
    hd.num_ctas = a.num_ctas;
    hd.max_splits = nsplit_of(Pmax, C);
    hd.tail_requests = tail_requests;
    hd.tail_chunk = tail_requests > 0 ? Ct : 0;
    hd.batch = a.B;
    hd.num_kv_heads = a.Hkv;
    hd.items_cap = a.items_cap;
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
  float* part_o;
  float* part_lse;
  int Hq, Hkv;
  float scale_log2;  // sm_scale * log2(e)
  int out_bf16;
};

struct __align__(16) SlotItem {  // item handed from the producer to the consumers
  WorkItem it;
  int idx, pad[3];
};

struct SmemLayout {
  static constexpr int stages = 0;
  static constexpr int qslots = stages + kStages * kStageBytes;
  static constexpr int items = qslots + kItemSlots * kQSlotBytes;
  static constexpr int merge_o = items + kItemSlots * (int)sizeof(SlotItem);
  static constexpr int merge_m = merge_o + kConsumerWarps * kMaxG * kMergeStride * 4;
  static constexpr int merge_l = merge_m + kConsumerWarps * kMaxG * 4;
  static constexpr int bars = merge_l + kConsumerWarps * kMaxG * 4;
  static constexpr int nbars = 2 * kStages + 2 * kItemSlots;
  static constexpr int flag = bars + nbars * 8;
  static constexpr int total = flag + 16;
  static constexpr int alloc = total + 1024;  // room to align the base to 1024 B (128B swizzle)
};
static_assert(kMaxSplits * kMaxG * 4 <= kConsumerWarps * kMaxG * kMergeStride * 4, "lse staging fits merge area");

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

// Byte offset of 16-B chunk cd (0..15) of token t in a staged slice: two
// 16-row x 128-B halves (d 0..63, d 64..127), 128-byte swizzle (chunk ^= row % 8).
__device__ __forceinline__ uint32_t slice_off(int t, int cd) {
  return (uint32_t)((cd >> 3) * kHalfBytes + t * 128 + (((cd & 7) ^ (t & 7)) << 4));
}

// One page (16 tokens) of one (request, kv head): S^T = K Q^T, online softmax, O^T += V^T P^T.
__device__ __forceinline__ void consume_page(uint32_t sbase, int valid, const uint32_t (&qf)[8][2],
                                             float (&acc)[8][4], float (&mrow)[2], float (&lrow)[2],
                                             float scale_log2, int lane) {
  using namespace dev;
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
      mma_bf16_16816(s, a0, a1, a2, a3, qf[kk][0], qf[kk][1]);
    }
  }
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
      mma_bf16_16816(acc[mt], a0, a1, a2, a3, bh0, bh1);
      mma_bf16_16816(acc[mt], a0, a1, a2, a3, bl0, bl1);
    }
  }
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

template <int G>
__global__ void __launch_bounds__(kThreads, 2)
    decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, RunArgs a) {
  using namespace dev;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  unsigned char* smem = smem_raw + ((1024u - (raw_u32 & 1023u)) & 1023u);
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + SmemLayout::bars;
  const uint32_t bar_empty = bar_full + kStages * 8;
  const uint32_t bar_ifull = bar_empty + kStages * 8;
  const uint32_t bar_iempty = bar_ifull + kItemSlots * 8;
  SlotItem* s_items = reinterpret_cast<SlotItem*>(smem + SmemLayout::items);
  float* merge_o = reinterpret_cast<float*>(smem + SmemLayout::merge_o);
  float* merge_m = reinterpret_cast<float*>(smem + SmemLayout::merge_m);
  float* merge_l = reinterpret_cast<float*>(smem + SmemLayout::merge_l);
  volatile int* s_flag = reinterpret_cast<volatile int*>(smem + SmemLayout::flag);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(bar_full + i * 8, 1);
      mbar_init(bar_empty + i * 8, 1);
    }
    for (int i = 0; i < kItemSlots; ++i) {
      mbar_init(bar_ifull + i * 8, 1);
      mbar_init(bar_iempty + i * 8, kConsumerWarps);
    }
    fence_mbar_init();
  }
  if (warp == kConsumerWarps && lane == 0) {
    prefetch_tmap(&tmK);
    prefetch_tmap(&tmV);
  }
  __syncthreads();
  // PDL: everything above overlapped the planner; the plan is read below.
  asm volatile("griddepcontrol.wait;" ::: "memory");

  const int n_items = a.header->n_items;
  const int W = gridDim.x;

  if (warp == kConsumerWarps) {
    // ============================== producer warp: items, Q and KV pages via TMA
    const uint64_t policy = policy_evict_first();
    bool exhausted = false;
    // Dynamic LPT scheduling: the first item is blockIdx.x, later ones come from
    // an atomic ticket (W + ticket) so idle CTAs take the next-largest item.
    auto draw = [&]() -> int {
      int idx = n_items;
      if (!exhausted) {
        int t = 0;
        if (lane == 0) t = atomicAdd(&a.header->sched_next, 1);
        idx = W + __shfl_sync(0xffffffffu, t, 0);
        if (idx >= n_items) {
          exhausted = true;
          idx = n_items;
          if (lane == 0) {
            const int done = atomicAdd(&a.header->sched_done, 1);
            if (done == W - 1) {  // every CTA stopped drawing: reset for the next run
              a.header->sched_next = 0;
              a.header->sched_done = 0;
            }
          }
        }
      }
      return idx;
    };
    int i_cur = blockIdx.x < n_items ? (int)blockIdx.x : n_items;
    int i_nxt = draw();
    WorkItem cur = load_item(a.items, i_cur, n_items);
    WorkItem nxt = load_item(a.items, i_nxt, n_items);
    int i_nn = draw();
    int cur_idx = (i_cur < n_items && lane < cur.pend - cur.pbeg) ? __ldg(a.indices + cur.pbeg + lane) : 0;
    uint32_t k = 0, qseq = 0;
    for (; i_cur < n_items; ++k) {
      // prefetch: the next item's first page ids, the item after's struct, one more ticket
      const int nxt_idx = (i_nxt < n_items && lane < nxt.pend - nxt.pbeg) ? __ldg(a.indices + nxt.pbeg + lane) : 0;
      const WorkItem nn = load_item(a.items, i_nn, n_items);
      const int i_nnn = draw();
      const uint32_t slot = k % kItemSlots;
      if (lane == 0) {
        mbar_wait(bar_iempty + slot * 8, ((k / kItemSlots) & 1) ^ 1);
        SlotItem si;
        si.it = cur;
        si.idx = i_cur;
        s_items[slot] = si;
        const uint32_t qbytes = G * kHeadDim * 2;
        mbar_arrive_expect_tx(bar_ifull + slot * 8, qbytes);
        bulk_load(sbase + SmemLayout::qslots + slot * kQSlotBytes,
                  a.q + ((size_t)cur.b * a.Hq + (size_t)cur.h * G) * kHeadDim, qbytes, bar_ifull + slot * 8);
      }
      const int np = cur.pend - cur.pbeg;
      int blk = cur_idx;
      for (int j0 = 0; j0 < np; j0 += 32) {
        const int nb = (j0 + 32 + lane < np) ? __ldg(a.indices + cur.pbeg + j0 + 32 + lane) : 0;
        const int cnt = min(32, np - j0);
        for (int j = 0; j < cnt; ++j) {
          const int page = __shfl_sync(0xffffffffu, blk, j);
          if (lane == 0) {
            const uint32_t st = qseq % kStages;
            mbar_wait(bar_empty + st * 8, ((qseq / kStages) & 1) ^ 1);
            const uint32_t fb = bar_full + st * 8;
            mbar_arrive_expect_tx(fb, kStageBytes);
            const int row = (page * a.Hkv + cur.h) * kPage;
            const uint32_t dst = sbase + SmemLayout::stages + st * kStageBytes;
            tma_load_3d(dst, &tmK, 0, row, 0, fb, policy);
            tma_load_3d(dst + kSliceBytes, &tmV, 0, row, 0, fb, policy);
          }
          ++qseq;
        }
        blk = nb;
      }
      i_cur = i_nxt;
      cur = nxt;
      cur_idx = nxt_idx;
      i_nxt = i_nn;
      nxt = nn;
      i_nn = i_nnn;
    }
    while (!exhausted) draw();  // make sure this CTA is counted as done
    // sentinel: tell the consumers there is no more work
    if (lane == 0) {
      const uint32_t slot = k % kItemSlots;
      mbar_wait(bar_iempty + slot * 8, ((k / kItemSlots) & 1) ^ 1);
      s_items[slot].it.b = -1;
      mbar_arrive(bar_ifull + slot * 8);
    }
    return;
  }

  // ============================== consumer warps
  const int g = lane >> 2, c = lane & 3;
  const int ct = threadIdx.x;  // 0..127
  uint32_t qbase = 0;
  for (uint32_t k = 0;; ++k) {
    const uint32_t slot = k % kItemSlots;
    mbar_wait(bar_ifull + slot * 8, (k / kItemSlots) & 1);
    const WorkItem it = s_items[slot].it;
    const int item_idx = s_items[slot].idx;
    if (it.b < 0) break;
    uint32_t qf[8][2];
    {
      const unsigned char* qs = smem + SmemLayout::qslots + slot * kQSlotBytes;
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
    __syncwarp();
    if (lane == 0) mbar_arrive(bar_iempty + slot * 8);

    float acc[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) acc[mt][0] = acc[mt][1] = acc[mt][2] = acc[mt][3] = 0.f;
    float mrow[2] = {-INFINITY, -INFINITY}, lrow[2] = {0.f, 0.f};
    const int np = it.pend - it.pbeg;
    for (int j = warp; j < np; j += kConsumerWarps) {
      const uint32_t q = qbase + j;
      const uint32_t st = q % kStages;
      mbar_wait(bar_full + st * 8, (q / kStages) & 1);
      const int valid = (j == np - 1) ? it.last_valid : kPage;
      consume_page(sbase + SmemLayout::stages + st * kStageBytes, valid, qf, acc, mrow, lrow, a.scale_log2, lane);
      __syncwarp();
      if (lane == 0) mbar_arrive(bar_empty + st * 8);
    }
    qbase += np;

    // ---- intra-CTA merge of the 4 warps' (m, l, O)
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      lrow[0] += __shfl_xor_sync(0xffffffffu, lrow[0], o);
      lrow[1] += __shfl_xor_sync(0xffffffffu, lrow[1], o);
    }
    {
      float* mo = merge_o + warp * (kMaxG * kMergeStride);
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
          sum += sc * merge_o[w * (kMaxG * kMergeStride) + head * kMergeStride + d];
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
    if (split) {
      // ---- a3: the last split of (b, kv head) to finish combines all splits.
      // Release: bar.sync orders every thread's partial stores before thread 0's
      // acq_rel ticket (cumulative); acquire: the ticket, then bar.sync, then reads.
      named_bar_sync(1, kConsumerThreads);
      if (ct == 0) {
        int* ctr = a.counters + (size_t)it.b * a.Hkv + it.h;
        const int old = atom_add_acq_rel_gpu(ctr, 1);
        const int last = (old == it.nsplit - 1);
        if (last) *ctr = 0;  // self-cleaning: ready for the next run with the same plan
        *s_flag = last;
      }
      named_bar_sync(1, kConsumerThreads);
      if (*s_flag) {
        float* s_lse = merge_o;  // reuse the merge area: [nsplit][G] base-2 lse
        const int ns = it.nsplit;
        for (int x = ct; x < ns * G; x += kConsumerThreads)
          s_lse[x] = __ldcg(a.part_lse + (size_t)it.part_base * G + x);
        named_bar_sync(1, kConsumerThreads);
#pragma unroll
        for (int o = ct; o < G * kHeadDim; o += kConsumerThreads) {
          const int head = o / kHeadDim, d = o % kHeadDim;
          float M = -INFINITY;
          for (int s = 0; s < ns; ++s) M = fmaxf(M, s_lse[s * G + head]);
          float sum = 0.f, L = 0.f;
          const float* po = a.part_o + ((size_t)it.part_base * G + head) * kHeadDim + d;
          int s = 0;
          for (; s + 8 <= ns; s += 8) {
            float v[8], w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(po + (size_t)(s + u) * G * kHeadDim);
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = ex2(s_lse[(s + u) * G + head] - M);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              sum += w[u] * v[u];
              L += w[u];
            }
          }
          for (; s < ns; ++s) {
            const float w = ex2(s_lse[s * G + head] - M);
            sum += w * __ldcg(po + (size_t)s * G * kHeadDim);
            L += w;
          }
          const size_t row = (size_t)it.b * a.Hq + (size_t)it.h * G + head;
          store_out(a, row * kHeadDim + d, sum / L);
          if (d == 0 && a.lse) a.lse[row] = (M + __log2f(L)) * kLn2;
        }
      }
    }
    named_bar_sync(1, kConsumerThreads);  // merge area free for the next item
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

template <int G>
l4_status launch_decode(const CUtensorMap& tk, const CUtensorMap& tv, const RunArgs& a, int grid, cudaStream_t st) {
  static bool attr_set[64] = {false};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 64 && !attr_set[dev]) {
    cudaError_t e = cudaFuncSetAttribute(decode_kernel<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, SmemLayout::alloc);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(decode_kernel<G>, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      cudaGetLastError();
      return L4_ERR_CUDA;
    }
    attr_set[dev] = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = SmemLayout::alloc;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL: overlap with the planner
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, decode_kernel<G>, tk, tv, a);
  if (e != cudaSuccess) {
    set_error("decode_kernel launch failed: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  return L4_OK;
}

l4_status device_ctas(int* ctas_out) {
  static int cache[64] = {0};
  int dev = 0;
  l4_status s = get_device(&dev);
  if (s != L4_OK) return s;
  if (dev < 64 && cache[dev] > 0) {
    *ctas_out = cache[dev];
    return L4_OK;
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
  if (dev < 64) cache[dev] = ctas;
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
  a.header = reinterpret_cast<PlanHeader*>(ws + L.header);
  a.items = reinterpret_cast<WorkItem*>(ws + L.items);
  a.counters = reinterpret_cast<int*>(ws + L.counters);
  const size_t smem = (size_t)5 * std::max(p->batch, 1) * sizeof(int);
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 5 * kMaxBatch * (int)sizeof(int));
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

static l4_status run_impl(const l4_decode_params* p, const void* q, const void* k_pages, const void* v_pages,
                          int64_t num_pages, const int32_t* page_indices, void* out, float* lse, void* workspace,
                          size_t workspace_bytes, cudaStream_t st) {
  int G = 0;
  l4_status s = check_params(p, &G);
  if (s != L4_OK) return s;
  if (p->batch == 0) return L4_OK;
  // page_indices may be NULL only when every request is empty (indptr[B] == 0).
  L4_CHECK_ARG(q && k_pages && v_pages && out, "q/k_pages/v_pages/out is NULL");
  L4_CHECK_ARG(num_pages >= 1, "num_pages must be >= 1");
  L4_CHECK_ARG((reinterpret_cast<uintptr_t>(q) & 15) == 0, "q must be 16-byte aligned");
  if (!workspace) return fail(L4_ERR_WORKSPACE, "workspace is NULL");
  WsLayout L;
  if (!ws_layout_from_bytes(p->batch, p->num_kv_heads, G, workspace_bytes, &L))
    return fail(L4_ERR_WORKSPACE, "workspace too small");
  int ctas = 0;
  s = device_ctas(&ctas);
  if (s != L4_OK) return s;
  const int64_t rows = num_pages * p->num_kv_heads * kPage;
  CUtensorMap tk, tv;
  s = make_tmap(&tk, k_pages, rows);
  if (s != L4_OK) return s;
  s = make_tmap(&tv, v_pages, rows);
  if (s != L4_OK) return s;
  char* ws = static_cast<char*>(workspace);
  RunArgs a;
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.out = out;
  a.lse = lse;
  a.indices = page_indices;
  a.items = reinterpret_cast<const WorkItem*>(ws + L.items);
  a.header = reinterpret_cast<PlanHeader*>(ws + L.header);
  a.counters = reinterpret_cast<int*>(ws + L.counters);
  a.part_o = reinterpret_cast<float*>(ws + L.part_o);
  a.part_lse = reinterpret_cast<float*>(ws + L.part_lse);
  a.Hq = p->num_q_heads;
  a.Hkv = p->num_kv_heads;
  const float scale = p->sm_scale > 0.f ? p->sm_scale : 1.0f / std::sqrt((float)kHeadDim);
  a.scale_log2 = scale * kLog2e;
  a.out_bf16 = p->out_dtype == L4_DT_BF16;
  switch (G) {
    case 1: return launch_decode<1>(tk, tv, a, ctas, st);
    case 2: return launch_decode<2>(tk, tv, a, ctas, st);
    case 4: return launch_decode<4>(tk, tv, a, ctas, st);
    default: return launch_decode<8>(tk, tv, a, ctas, st);
  }
}

extern "C" l4_status l4_decode_plan(const l4_decode_params* p, const int32_t* kv_len, const int32_t* page_indptr,
                                    int64_t total_pages, void* workspace, size_t workspace_bytes, void* stream) {
  if (p && p->batch == 0) {
    int G = 0;
    return check_params(p, &G);
  }
  return plan_impl(p, kv_len, page_indptr, total_pages, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" l4_status l4_decode_run(const l4_decode_params* p, const void* q, const void* k_pages, const void* v_pages,
                                   int64_t num_pages, const int32_t* page_indices, void* out, float* lse,
                                   void* workspace, size_t workspace_bytes, void* stream) {
  return run_impl(p, q, k_pages, v_pages, num_pages, page_indices, out, lse, workspace, workspace_bytes,
                  static_cast<cudaStream_t>(stream));
}

extern "C" l4_status l4_decode_attention(const l4_decode_params* p, const void* q, const void* k_pages,
                                         const void* v_pages, int64_t num_pages, const int32_t* page_indptr,
                                         const int32_t* page_indices, int64_t total_pages, const int32_t* kv_len,
                                         void* out, float* lse, void* workspace, size_t workspace_bytes,
                                         void* stream) {
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

extern "C" l4_status l4_decode_plan_items(const void* workspace, int32_t* items_out, int32_t max_items, void* stream) {
  L4_CHECK_ARG(workspace && items_out && max_items >= 0, "bad arguments");
  PlanHeader h;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = cudaMemcpyAsync(&h, workspace, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    const size_t items_off = align256(256 + (size_t)std::max(h.batch, 1) * h.num_kv_heads * sizeof(int));
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
