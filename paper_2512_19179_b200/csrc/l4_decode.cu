// l4_decode: length-binned split-KV GQA decode attention over a paged KV cache,
// for B200 (sm_100a).  Entry points: l4_decode_workspace_size / _plan / _run /
// _attention in include/l4.h.
//
// What is computed (definition in oracle/attention.py): for
// every request b and q-head h, softmax(scale * q K^T) V over the L_b cached
// tokens of kv head h/G, plus the natural-log LSE.
//
// How (B200 design):
//  a1  plan_kernel (1 CTA): pages -> chunk size C -> near-equal splits per
//      request -> items binned by chunk length, longest bin first (LPT), so the
//      longest request's splits start first and short requests fill the tail
//      (the paper's inter-SM imbalance).  Zeroes split counters.
//  a2  decode_kernel (persistent, 1 producer + 4 consumer warps per CTA):
//      the producer warp streams each (page, kv head) K and V slice (4 KB each,
//      HND layout) with TMA (cp.async.bulk.tensor, 128B swizzle, L2
//      evict-first) into an 8-stage shared-memory ring tracked by mbarriers;
//      consumer warps compute S^T = K Q^T and O^T += V^T P^T with mma.sync
//      m16n8k16 (tokens / head_dim on the M side, the G <= 8 query heads on
//      the N side, so GQA group 8 has no padding), an online softmax with
//      warp-shuffle max reductions in the exp2 domain, and P split into
//      bf16 hi + lo (reading Z23) so the probability rounding stays < 1e-5.
//  a3  LSE combine: the 4 warps of a CTA merge their (m, l, O) in shared
//      memory; a split item writes (O/l, lse) to the workspace and the last
//      split to finish for (b, kv head) (atomic counter) combines all splits
//      (FlashDecoding aggregation) — no second kernel launch.
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
constexpr int kThreads = (kConsumerWarps + 1) * 32;  // 160
constexpr int kStages = 8;
constexpr int kTileBytes = kPage * 64 * 2;            // 16 rows x 64 bf16 = 2 KB (one 128B-swizzle box)
constexpr int kStageBytes = 4 * kTileBytes;           // K[0:64], K[64:128], V[0:64], V[64:128]
constexpr int kItemSlots = 4;
constexpr int kMaxG = 8;
constexpr int kQSlotBytes = kMaxG * kHeadDim * 2;     // 2 KB
constexpr int kMergeStride = kHeadDim + 4;            // floats per head row (bank-conflict padding)
constexpr int kMaxSplits = 512;                       // per (request, kv head); lse staging capacity
constexpr int kMinChunk = 8;                          // pages
constexpr int kItemsPerCta = 8;                       // auto chunk target
constexpr int kMaxBatch = 8192;
constexpr int kPlanThreads = 1024;
constexpr int kNumBins = 32;
constexpr float kLn2 = 0.69314718055994530942f;
constexpr float kLog2e = 1.44269504088896340736f;

struct __align__(16) WorkItem {
  int b, h, pbeg, pend, last_valid, part_base, nsplit, split;
};
static_assert(sizeof(WorkItem) == 32, "WorkItem is 32 bytes");

struct __align__(16) PlanHeader {
  int n_items, chunk, num_ctas, max_splits;
  int batch, num_kv_heads, items_cap, pad;
  int pad2[8];
};
static_assert(sizeof(PlanHeader) == 64, "PlanHeader is 64 bytes");

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

// ------------------------------------------------------------------ device info cache
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

int num_ctas_for(int sms, int occ) { return sms * std::max(1, std::min(occ, 2)); }

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

// items_cap: upper bound on work items for any batch with <= max_total_pages pages.
int items_cap_for(const l4_decode_params* p, int64_t max_total_pages, int num_ctas) {
  const int64_t B = p->batch, Hkv = p->num_kv_heads;
  int64_t cap;
  if (p->chunk_pages < 0) {
    cap = B * Hkv;
  } else if (p->chunk_pages > 0) {
    cap = Hkv * (B + ceil_div64(max_total_pages, p->chunk_pages));
  } else {
    cap = std::min(Hkv * (B + ceil_div64(max_total_pages, kMinChunk)),
                   Hkv * B + (int64_t)num_ctas * kItemsPerCta + Hkv);
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

__device__ __forceinline__ int warp_incl_scan(int v) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) >= o) v += t;
  }
  return v;
}

// Block-wide exclusive scan of one int per thread (1024 threads); returns the
// exclusive prefix and the block total.
__device__ int block_excl_scan(int v, int* total, int* s_warp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = warp_incl_scan(v);
  __syncthreads();
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = s_warp[lane];
    int wi = warp_incl_scan(w);
    s_warp[lane] = wi - w;
    if (lane == 31) s_warp[32] = wi;
  }
  __syncthreads();
  *total = s_warp[32];
  return s_warp[warp] + incl - v;
}

__device__ long long block_sum_ll(long long v, long long* s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) s[warp] = v;
  __syncthreads();
  long long t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += s[i];
  return t;
}

__device__ int block_max_i(int v, int* s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  if (lane == 0) s[warp] = v;
  __syncthreads();
  int t = 0;
  for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t = max(t, s[i]);
  return t;
}

__device__ __forceinline__ int nsplit_of(int pages, long long C) {
  if (pages <= 0) return 1;
  return (int)((pages + C - 1) / C);
}

__device__ __forceinline__ int bin_of(int pages, int nsplit) {
  if (pages <= 0) return 0;
  const int ip = (pages + nsplit - 1) / nsplit;  // pages of the largest split
  return min(kNumBins - 1, 32 - __clz(ip));      // bit_length(ip)
}

constexpr int kPlanMaxR = kMaxBatch / kPlanThreads;  // requests per thread

__global__ void __launch_bounds__(kPlanThreads, 1) plan_kernel(PlanArgs a) {
  extern __shared__ int plan_smem[];          // s_off[B], s_b[B] (binned order)
  int* s_off = plan_smem;
  int* s_b = plan_smem + max(a.B, 1);
  __shared__ long long s_ll[32];
  __shared__ int s_i[33];
  __shared__ int s_hist[kNumBins];
  const int tid = threadIdx.x;
  const int R = (a.B + kPlanThreads - 1) / kPlanThreads;

  int pages[kPlanMaxR];
  long long my_sum = 0;
  int my_max = 0;
#pragma unroll
  for (int r = 0; r < kPlanMaxR; ++r) {
    const int b = tid * R + r;
    int pg = 0;
    if (r < R && b < a.B) {
      const int L = a.kv_len[b];
      pg = L > 0 ? (L + kPage - 1) / kPage : 0;
    }
    pages[r] = pg;
    my_sum += pg;
    my_max = max(my_max, pg);
  }
  const long long T = block_sum_ll(my_sum, s_ll);
  const int Pmax = block_max_i(my_max, s_i);

  // chunk size C (pages per work item)
  long long C;
  if (a.forced_chunk > 0) {
    C = a.forced_chunk;
  } else if (a.forced_chunk < 0) {
    C = (long long)INT_MAX;
  } else {
    const long long denom = (long long)a.num_ctas * kItemsPerCta;
    C = max((long long)kMinChunk, (T * a.Hkv + denom - 1) / denom);
  }
  C = max(C, (long long)((Pmax + kMaxSplits - 1) / kMaxSplits));
  long long N;
  for (;;) {  // grow C until the work list fits the workspace (block-uniform loop)
    long long my_items = 0;
#pragma unroll
    for (int r = 0; r < kPlanMaxR; ++r)
      if (r < R && tid * R + r < a.B) my_items += (long long)nsplit_of(pages[r], C) * a.Hkv;
    N = block_sum_ll(my_items, s_ll);
    if (N <= a.items_cap) break;
    C *= 2;
  }

  // ---- length bins, longest first (stable by request index within a bin)
  if (tid < kNumBins) s_hist[tid] = 0;
  __syncthreads();
  int bins[kPlanMaxR];
#pragma unroll
  for (int r = 0; r < kPlanMaxR; ++r) {
    const bool valid = r < R && tid * R + r < a.B;
    bins[r] = valid ? bin_of(pages[r], nsplit_of(pages[r], C)) : -1;
    if (valid) atomicAdd(&s_hist[bins[r]], 1);
  }
  __syncthreads();
  int base_items = 0, base_rank = 0;
  for (int bin = kNumBins - 1; bin >= 0; --bin) {
    if (s_hist[bin] == 0) continue;  // block-uniform
    int my_cnt = 0, my_n = 0;
#pragma unroll
    for (int r = 0; r < kPlanMaxR; ++r)
      if (bins[r] == bin) {
        my_cnt += nsplit_of(pages[r], C) * a.Hkv;
        my_n += 1;
      }
    int tot_items, tot_n;
    const int ex_items = block_excl_scan(my_cnt, &tot_items, s_i);
    const int ex_n = block_excl_scan(my_n, &tot_n, s_i);
    int off = base_items + ex_items, rank = base_rank + ex_n;
#pragma unroll
    for (int r = 0; r < kPlanMaxR; ++r)
      if (bins[r] == bin) {
        s_off[rank] = off;
        s_b[rank] = tid * R + r;
        off += nsplit_of(pages[r], C) * a.Hkv;
        rank += 1;
      }
    base_items += tot_items;
    base_rank += tot_n;
  }
  __syncthreads();

  // ---- write the items cooperatively: item i -> request by binary search over s_off
  const int nreq = a.B;
  for (int i = tid; i < (int)N; i += kPlanThreads) {
    int lo = 0, hi = nreq - 1;
    while (lo < hi) {  // last rank with s_off[rank] <= i
      const int mid = (lo + hi + 1) >> 1;
      if (s_off[mid] <= i) lo = mid; else hi = mid - 1;
    }
    const int b = s_b[lo];
    const int L = a.kv_len[b];
    const int pg = L > 0 ? (L + kPage - 1) / kPage : 0;
    const int ns = nsplit_of(pg, C);
    const int local = i - s_off[lo];
    const int h = local / ns, s = local - h * ns;
    const int p0 = (int)(((long long)s * pg) / ns);
    const int p1 = (int)(((long long)(s + 1) * pg) / ns);
    const int base = a.indptr[b];
    WorkItem it;
    it.b = b;
    it.h = h;
    it.pbeg = base + p0;
    it.pend = base + p1;
    it.last_valid = (p1 == pg && pg > 0) ? (L - (pg - 1) * kPage) : (p1 > p0 ? kPage : 0);
    it.part_base = s_off[lo] + h * ns;
    it.nsplit = ns;
    it.split = s;
    a.items[i] = it;
  }
  for (int i = tid; i < a.B * a.Hkv; i += kPlanThreads) a.counters[i] = 0;
  if (tid == 0) {
    PlanHeader hd;
    memset(&hd, 0, sizeof(hd));
    hd.n_items = (int)N;
    hd.chunk = (int)min(C, (long long)INT_MAX);
    hd.num_ctas = a.num_ctas;
    hd.max_splits = nsplit_of(Pmax, C);
    hd.batch = a.B;
    hd.num_kv_heads = a.Hkv;
    hd.items_cap = a.items_cap;
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
  const PlanHeader* header;
  int* counters;
  float* part_o;
  float* part_lse;
  int Hq, Hkv;
  float scale_log2;  // sm_scale * log2(e)
  int out_bf16;
};

struct SmemLayout {
  static constexpr int stages = 0;
  static constexpr int qslots = stages + kStages * kStageBytes;
  static constexpr int items = qslots + kItemSlots * kQSlotBytes;
  static constexpr int merge_o = items + kItemSlots * (int)sizeof(WorkItem);
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
    const uint32_t row = sbase + tok * 128;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int cd = kk * 2 + (mi >> 1);  // 16-B chunk 0..15 of the 256-B row
      const uint32_t addr = row + (cd >> 3) * kTileBytes + (((cd & 7) ^ r8) << 4);
      uint32_t a0, a1, a2, a3;
      ldmatrix_x4(addr, a0, a1, a2, a3);
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
    const uint32_t row = sbase + 2 * kTileBytes + tok * 128;
    // masks for invalid tokens of a partial last page (V may hold NaN there)
    const uint32_t mlo = (((2 * c) < valid) ? 0x0000ffffu : 0u) | (((2 * c + 1) < valid) ? 0xffff0000u : 0u);
    const uint32_t mhi = (((2 * c + 8) < valid) ? 0x0000ffffu : 0u) | (((2 * c + 9) < valid) ? 0xffff0000u : 0u);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const int cd = mt * 2 + (mi & 1);
      const uint32_t addr = row + (cd >> 3) * kTileBytes + (((cd & 7) ^ r8) << 4);
      uint32_t a0, a1, a2, a3;
      ldmatrix_x4_trans(addr, a0, a1, a2, a3);
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

template <int G>
__global__ void __launch_bounds__(kThreads, 2)
    decode_kernel(const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmV, RunArgs a) {
  using namespace dev;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t sbase = smem_u32(smem);
  const uint32_t bar_full = sbase + SmemLayout::bars;
  const uint32_t bar_empty = bar_full + kStages * 8;
  const uint32_t bar_ifull = bar_empty + kStages * 8;
  const uint32_t bar_iempty = bar_ifull + kItemSlots * 8;
  WorkItem* s_items = reinterpret_cast<WorkItem*>(smem + SmemLayout::items);
  float* merge_o = reinterpret_cast<float*>(smem + SmemLayout::merge_o);
  float* merge_m = reinterpret_cast<float*>(smem + SmemLayout::merge_m);
  float* merge_l = reinterpret_cast<float*>(smem + SmemLayout::merge_l);
  int* s_flag = reinterpret_cast<int*>(smem + SmemLayout::flag);

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
  __syncthreads();

  const int n_items = a.header->n_items;
  const int W = gridDim.x;

  if (warp == kConsumerWarps) {
    // ============================== producer warp: items, Q and KV pages via TMA
    if (lane == 0) {
      prefetch_tmap(&tmK);
      prefetch_tmap(&tmV);
    }
    const uint64_t policy = policy_evict_first();
    auto load_item = [&](int i) -> WorkItem {
      WorkItem it;
      if (i < n_items) {
        const int4* p = reinterpret_cast<const int4*>(a.items + i);
        int4 x = __ldg(p), y = __ldg(p + 1);
        it.b = x.x; it.h = x.y; it.pbeg = x.z; it.pend = x.w;
        it.last_valid = y.x; it.part_base = y.y; it.nsplit = y.z; it.split = y.w;
      } else {
        it.b = 0; it.h = 0; it.pbeg = 0; it.pend = 0; it.last_valid = 0; it.part_base = 0; it.nsplit = 1; it.split = 0;
      }
      return it;
    };
    int i = blockIdx.x;
    WorkItem cur = load_item(i);
    WorkItem nxt = load_item(i + W);
    int cur_idx = (i < n_items && lane < cur.pend - cur.pbeg) ? __ldg(a.indices + cur.pbeg + lane) : 0;
    uint32_t k = 0;
    uint32_t qseq = 0;
    for (; i < n_items; i += W, ++k) {
      const WorkItem nn = load_item(i + 2 * W);
      const int nxt_idx = (i + W < n_items && lane < nxt.pend - nxt.pbeg) ? __ldg(a.indices + nxt.pbeg + lane) : 0;
      const uint32_t slot = k % kItemSlots;
      if (lane == 0) {
        mbar_wait(bar_iempty + slot * 8, ((k / kItemSlots) & 1) ^ 1);
        s_items[slot] = cur;
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
            tma_load_2d(dst, &tmK, 0, row, fb, policy);
            tma_load_2d(dst + kTileBytes, &tmK, 64, row, fb, policy);
            tma_load_2d(dst + 2 * kTileBytes, &tmV, 0, row, fb, policy);
            tma_load_2d(dst + 3 * kTileBytes, &tmV, 64, row, fb, policy);
          }
          ++qseq;
        }
        blk = nb;
      }
      cur = nxt;
      nxt = nn;
      cur_idx = nxt_idx;
    }
    return;
  }

  // ============================== consumer warps
  const int g = lane >> 2, c = lane & 3;
  const int ct = threadIdx.x;  // 0..127
  uint32_t k = 0;
  uint32_t qbase = 0;
  for (int i = blockIdx.x; i < n_items; i += W, ++k) {
    const uint32_t slot = k % kItemSlots;
    mbar_wait(bar_ifull + slot * 8, (k / kItemSlots) & 1);
    const WorkItem it = s_items[slot];
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
    named_bar_sync(1, kConsumerWarps * 32);
    const bool split = it.nsplit > 1;
#pragma unroll
    for (int o = ct; o < G * kHeadDim; o += kConsumerWarps * 32) {
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
        const size_t prow = (size_t)i * G + head;  // partial slot = item index
        a.part_o[prow * kHeadDim + d] = val;
        if (d == 0) a.part_lse[prow] = lse2;
      }
    }
    if (split) {
      // ---- a3: the last split of (b, kv head) to finish combines all splits
      __threadfence();
      named_bar_sync(1, kConsumerWarps * 32);
      if (ct == 0) {
        int* ctr = a.counters + (size_t)it.b * a.Hkv + it.h;
        const int old = atomicAdd(ctr, 1);
        const int last = (old == it.nsplit - 1);
        if (last) *ctr = 0;  // self-cleaning: ready for the next run with the same plan
        *s_flag = last;
      }
      named_bar_sync(1, kConsumerWarps * 32);
      if (*s_flag) {
        __threadfence();
        float* s_lse = merge_o;  // reuse the merge area: [nsplit][G] base-2 lse
        const int ns = it.nsplit;
        for (int x = ct; x < ns * G; x += kConsumerWarps * 32)
          s_lse[x] = __ldcg(a.part_lse + (size_t)it.part_base * G + x);
        named_bar_sync(1, kConsumerWarps * 32);
#pragma unroll
        for (int o = ct; o < G * kHeadDim; o += kConsumerWarps * 32) {
          const int head = o / kHeadDim, d = o % kHeadDim;
          float M = -INFINITY;
          for (int s = 0; s < ns; ++s) M = fmaxf(M, s_lse[s * G + head]);
          float sum = 0.f, L = 0.f;
          const float* po = a.part_o + ((size_t)it.part_base * G + head) * kHeadDim + d;
          int s = 0;
          for (; s + 4 <= ns; s += 4) {
            const float v0 = __ldcg(po + (size_t)(s + 0) * G * kHeadDim);
            const float v1 = __ldcg(po + (size_t)(s + 1) * G * kHeadDim);
            const float v2 = __ldcg(po + (size_t)(s + 2) * G * kHeadDim);
            const float v3 = __ldcg(po + (size_t)(s + 3) * G * kHeadDim);
            const float w0 = ex2(s_lse[(s + 0) * G + head] - M), w1 = ex2(s_lse[(s + 1) * G + head] - M);
            const float w2 = ex2(s_lse[(s + 2) * G + head] - M), w3 = ex2(s_lse[(s + 3) * G + head] - M);
            sum += w0 * v0 + w1 * v1 + w2 * v2 + w3 * v3;
            L += (w0 + w1) + (w2 + w3);
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
    named_bar_sync(1, kConsumerWarps * 32);  // merge area free for the next item
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

// Pool [num_pages, Hkv, 16, 128] bf16 viewed as a 2-D tensor of num_pages*Hkv*16
// rows x 128 columns; box = 16 rows x 64 columns (128 B), 128-byte swizzle.
l4_status make_tmap(CUtensorMap* tm, const void* base, int64_t rows) {
  auto enc = get_encode_fn();
  if (!enc) return fail(L4_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (driver too old or no device)");
  if (rows <= 0 || rows > ((int64_t)1 << 32)) return fail(L4_ERR_INVALID_ARG, "KV pool too large for a tensor map");
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return fail(L4_ERR_INVALID_ARG, "KV pool must be 16-byte aligned");
  cuuint64_t dims[2] = {(cuuint64_t)kHeadDim, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kHeadDim * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)kPage};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
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
    if (e != cudaSuccess) {
      set_error("cudaFuncSetAttribute: %s", cudaGetErrorString(e));
      cudaGetLastError();
      return L4_ERR_CUDA;
    }
    attr_set[dev] = true;
  }
  decode_kernel<G><<<grid, kThreads, SmemLayout::alloc, st>>>(tk, tv, a);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("decode_kernel launch failed: %s", cudaGetErrorString(e));
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
  // Two persistent CTAs per SM (each ~92 KB of shared memory, 160 threads).
  const int ctas = num_ctas_for(sms, 2);
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
  const size_t smem = (size_t)2 * std::max(p->batch, 1) * sizeof(int);
  static std::once_flag once;
  std::call_once(once, [] {
    cudaFuncSetAttribute(plan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kMaxBatch * (int)sizeof(int));
  });
  plan_kernel<<<1, kPlanThreads, smem, st>>>(a);
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
  L4_CHECK_ARG(q && k_pages && v_pages && out && page_indices, "q/k_pages/v_pages/out/page_indices is NULL");
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
  a.header = reinterpret_cast<const PlanHeader*>(ws + L.header);
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
