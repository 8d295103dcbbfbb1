// l4_migrate / l4_copy_pages / l4_pack_pages / l4_unpack_pages and CUDA IPC helpers.
//
// P:281  "allocates memory on the target instance, and transfers the KV cache"
// P:426  intra-node transfers with cudaMemcpyPeerAsync, avoiding NCCL
//        collectives that are "ill-suited for numerous small messages"
// P:428  "KV caches are transferred directly into idle slots on the target
//        instance, and migration is skipped if no idle cache is available."
//
// B200 design: one SM-driven copy kernel per call moves every (page, layer,
// K|V) slice with 16-byte vector loads from the source pool and 16-byte
// stores straight into the destination slots — local, peer (P2P over
// NVLink 5 / NVSwitch) or CUDA-IPC-mapped memory of another process — so a
// request of thousands of 32 KB page slices costs one launch, not thousands
// of cudaMemcpyPeerAsync calls.  The grid is capped at 2 CTAs per SM so that a
// concurrent decode kernel keeps most of the machine.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <vector>

#include "l4_internal.h"

namespace l4 {
namespace {

constexpr int kPairsPerLaunch = 1024;  // page pairs carried in the kernel parameters (8 KB)
constexpr int kCopyThreads = 256;

// One side of a copy: a paged pool (mode 0) or a contiguous staging buffer (mode 1).
struct Side {
  char* k;
  char* v;
  long long layer_stride;
  int mode;
};

struct CopyArgs {
  Side src, dst;
  long long page_bytes;  // multiple of 16
  int layers;
  int n;                 // pairs in this launch
  long long stage_base;  // index of the first pair within the whole staging buffer
  int src_page[kPairsPerLaunch];
  int dst_page[kPairsPerLaunch];
};

__device__ __forceinline__ char* slice_addr(const Side& s, int page, long long pair_index, int layer, int kv,
                                            long long page_bytes, int layers) {
  if (s.mode == 0) return (kv ? s.v : s.k) + (long long)layer * s.layer_stride + (long long)page * page_bytes;
  return s.k + (((pair_index * layers) + layer) * 2 + kv) * page_bytes;
}

// One CTA iteration copies one whole (page, layer, K|V) slice: the slice index is decoded once,
// then every thread moves kUnroll 16-byte chunks with all loads issued before the stores.
constexpr int kUnroll = 8;
__global__ void __launch_bounds__(kCopyThreads) copy_pages_kernel(const __grid_constant__ CopyArgs a) {
  const long long chunks = a.page_bytes >> 4;  // 16-byte units per slice
  const long long slices = (long long)a.n * a.layers * 2;
  for (long long sl = blockIdx.x; sl < slices; sl += gridDim.x) {
    const int kv = (int)(sl & 1);
    const long long pl = sl >> 1;
    const int layer = (int)(pl % a.layers);
    const int i = (int)(pl / a.layers);
    const int4* src = reinterpret_cast<const int4*>(
        slice_addr(a.src, a.src_page[i], a.stage_base + i, layer, kv, a.page_bytes, a.layers));
    int4* dst = reinterpret_cast<int4*>(slice_addr(a.dst, a.dst_page[i], a.stage_base + i, layer, kv, a.page_bytes, a.layers));
    for (long long c0 = threadIdx.x; c0 < chunks; c0 += (long long)kCopyThreads * kUnroll) {
      int4 v[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const long long c = c0 + (long long)u * kCopyThreads;
        if (c < chunks) v[u] = __ldcs(src + c);
      }
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const long long c = c0 + (long long)u * kCopyThreads;
        if (c < chunks) __stcs(dst + c, v[u]);
      }
    }
  }
}

l4_status check_view(const l4_kv_view* v, const char* what) {
  if (!v) {
    set_error("%s view is NULL", what);
    return L4_ERR_INVALID_ARG;
  }
  if (!v->k_pages || !v->v_pages || v->num_pages < 0 || v->num_layers < 1 || v->page_bytes <= 0 ||
      (v->page_bytes & 15) || ((reinterpret_cast<uintptr_t>(v->k_pages) | reinterpret_cast<uintptr_t>(v->v_pages)) & 15)) {
    set_error("%s view invalid (NULL pools, layers < 1, or page_bytes / pointers not 16-byte aligned)", what);
    return L4_ERR_INVALID_ARG;
  }
  if (v->num_layers > 1 && v->layer_stride_bytes < v->num_pages * v->page_bytes) {
    set_error("%s view: layer_stride_bytes < num_pages * page_bytes", what);
    return L4_ERR_INVALID_ARG;
  }
  return L4_OK;
}

l4_status check_pages(const int32_t* pages, int64_t n, int64_t num_pages, const char* what) {
  for (int64_t i = 0; i < n; ++i)
    if (pages[i] < 0 || pages[i] >= num_pages) {
      set_error("%s page id %d out of range [0, %lld)", what, (int)pages[i], (long long)num_pages);
      return L4_ERR_INVALID_ARG;
    }
  return L4_OK;
}

int copy_grid(long long slices) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (int)std::max<long long>(1, std::min<long long>(slices, 2LL * sms));  // <= 2 CTAs per SM
}

l4_status launch_copies(const Side& src, const Side& dst, long long page_bytes, int layers, const int32_t* sp,
                        const int32_t* dp, int64_t n, cudaStream_t st) {
  for (int64_t off = 0; off < n; off += kPairsPerLaunch) {
    CopyArgs a;
    std::memset(&a, 0, sizeof(a));
    a.src = src;
    a.dst = dst;
    a.page_bytes = page_bytes;
    a.layers = layers;
    a.n = (int)std::min<int64_t>(kPairsPerLaunch, n - off);
    a.stage_base = off;
    for (int i = 0; i < a.n; ++i) {
      a.src_page[i] = sp ? sp[off + i] : 0;
      a.dst_page[i] = dp ? dp[off + i] : 0;
    }
    copy_pages_kernel<<<copy_grid((long long)a.n * layers * 2), kCopyThreads, 0, st>>>(a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("copy_pages_kernel launch failed: %s", cudaGetErrorString(e));
      return L4_ERR_CUDA;
    }
  }
  return L4_OK;
}

Side pool_side(const l4_kv_view* v) {
  Side s;
  s.k = static_cast<char*>(v->k_pages);
  s.v = static_cast<char*>(v->v_pages);
  s.layer_stride = v->layer_stride_bytes;
  s.mode = 0;
  return s;
}

}  // namespace
}  // namespace l4

using namespace l4;

extern "C" l4_status l4_copy_pages(const l4_kv_view* src, const int32_t* src_pages, const l4_kv_view* dst,
                                   const int32_t* dst_pages, int64_t n_pages, void* stream) {
  NvtxRange nvtx("l4_copy_pages");
  l4_status s = check_view(src, "src");
  if (s != L4_OK) return s;
  s = check_view(dst, "dst");
  if (s != L4_OK) return s;
  L4_CHECK_ARG(n_pages >= 0, "n_pages < 0");
  L4_CHECK_ARG(n_pages == 0 || (src_pages && dst_pages), "page lists are NULL");
  L4_CHECK_ARG(src->page_bytes == dst->page_bytes && src->num_layers == dst->num_layers,
               "src and dst views differ in page_bytes or num_layers");
  if ((s = check_pages(src_pages, n_pages, src->num_pages, "src")) != L4_OK) return s;
  if ((s = check_pages(dst_pages, n_pages, dst->num_pages, "dst")) != L4_OK) return s;
  if (n_pages == 0) return L4_OK;
  return launch_copies(pool_side(src), pool_side(dst), src->page_bytes, src->num_layers, src_pages, dst_pages, n_pages,
                       static_cast<cudaStream_t>(stream));
}

extern "C" l4_status l4_migrate(const l4_kv_view* src, const int32_t* src_pages, int64_t n_pages,
                                const l4_kv_view* dst, l4_page_pool* dst_pool, int32_t* dst_pages_out, void* stream,
                                void* done_event) {
  NvtxRange nvtx("l4_migrate");
  l4_status s = check_view(src, "src");
  if (s != L4_OK) return s;
  s = check_view(dst, "dst");
  if (s != L4_OK) return s;
  L4_CHECK_ARG(dst_pool != nullptr, "dst_pool is NULL");
  L4_CHECK_ARG(n_pages >= 0, "n_pages < 0");
  L4_CHECK_ARG(n_pages == 0 || (src_pages && dst_pages_out), "page lists are NULL");
  L4_CHECK_ARG(src->page_bytes == dst->page_bytes && src->num_layers == dst->num_layers,
               "src and dst views differ in page_bytes or num_layers");
  if ((s = check_pages(src_pages, n_pages, src->num_pages, "src")) != L4_OK) return s;
  std::vector<int32_t> dp((size_t)n_pages);
  s = l4_pool_alloc(dst_pool, n_pages, dp.data());  // all-or-nothing; NO_PAGES leaves the pool unchanged
  if (s != L4_OK) return s;
  for (int64_t i = 0; i < n_pages; ++i)
    if (dp[(size_t)i] >= dst->num_pages) {
      l4_pool_free(dst_pool, dp.data(), n_pages);
      return fail(L4_ERR_INVALID_ARG, "dst_pool has more pages than the dst view");
    }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n_pages > 0) {
    s = launch_copies(pool_side(src), pool_side(dst), src->page_bytes, src->num_layers, src_pages, dp.data(), n_pages,
                      st);
    if (s != L4_OK) {
      // launch_copies enqueues one kernel per kPairsPerLaunch pages: chunks launched before the
      // failing one still write into the destination pages, so wait for them before the pages
      // go back to the pool (a failed synchronisation keeps them allocated: never reused while
      // a copy may still land, and their ids are reported)
      if (cudaStreamSynchronize(st) == cudaSuccess) {
        l4_pool_free(dst_pool, dp.data(), n_pages);
      } else {
        cudaGetLastError();
        std::memcpy(dst_pages_out, dp.data(), (size_t)n_pages * sizeof(int32_t));
      }
      return s;
    }
  }
  // the destination ids are the caller's from here on, even if recording the event fails
  std::memcpy(dst_pages_out, dp.data(), (size_t)n_pages * sizeof(int32_t));
  if (done_event) {
    cudaError_t e = cudaEventRecord(static_cast<cudaEvent_t>(done_event), st);
    if (e != cudaSuccess) {
      set_error("cudaEventRecord: %s", cudaGetErrorString(e));
      cudaGetLastError();
      return L4_ERR_CUDA;  // the copy is enqueued; dst_pages_out holds the (allocated) pages
    }
  }
  return L4_OK;
}

extern "C" l4_status l4_pack_pages(const l4_kv_view* src, const int32_t* pages, int64_t n, void* staging,
                                   void* stream) {
  l4_status s = check_view(src, "src");
  if (s != L4_OK) return s;
  L4_CHECK_ARG(n >= 0 && (n == 0 || (pages && staging)), "bad page list / staging");
  L4_CHECK_ARG((reinterpret_cast<uintptr_t>(staging) & 15) == 0, "staging must be 16-byte aligned");
  if ((s = check_pages(pages, n, src->num_pages, "src")) != L4_OK) return s;
  if (n == 0) return L4_OK;
  Side d;
  d.k = static_cast<char*>(staging);
  d.v = nullptr;
  d.layer_stride = 0;
  d.mode = 1;
  return launch_copies(pool_side(src), d, src->page_bytes, src->num_layers, pages, nullptr, n,
                       static_cast<cudaStream_t>(stream));
}

extern "C" l4_status l4_unpack_pages(const l4_kv_view* dst, const int32_t* pages, int64_t n, const void* staging,
                                     void* stream) {
  l4_status s = check_view(dst, "dst");
  if (s != L4_OK) return s;
  L4_CHECK_ARG(n >= 0 && (n == 0 || (pages && staging)), "bad page list / staging");
  L4_CHECK_ARG((reinterpret_cast<uintptr_t>(staging) & 15) == 0, "staging must be 16-byte aligned");
  if ((s = check_pages(pages, n, dst->num_pages, "dst")) != L4_OK) return s;
  if (n == 0) return L4_OK;
  Side src;
  src.k = const_cast<char*>(static_cast<const char*>(staging));
  src.v = nullptr;
  src.layer_stride = 0;
  src.mode = 1;
  return launch_copies(src, pool_side(dst), dst->page_bytes, dst->num_layers, nullptr, pages, n,
                       static_cast<cudaStream_t>(stream));
}

namespace {
// cuMemGetAddressRange through the runtime's driver entry point (no libcuda link dependency).
typedef int (*PFN_getAddressRange)(unsigned long long*, size_t*, unsigned long long);
PFN_getAddressRange address_range_fn() {
  static PFN_getAddressRange fn = nullptr;
  static std::once_flag once;  // first calls from several host threads are safe
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_getAddressRange>(p);
    cudaGetLastError();
  });
  return fn;
}
}  // namespace

extern "C" l4_status l4_ipc_get_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
  L4_CHECK_ARG(dev_ptr && handle_out, "NULL argument");
  // The handle names the whole allocation that contains dev_ptr (a caching allocator such as
  // PyTorch's sub-allocates): report dev_ptr's offset from the allocation base, which is what
  // l4_ipc_open_handle maps in the other process.
  int64_t off = 0;
  if (offset_out) {
    auto fn = address_range_fn();
    unsigned long long base = 0;
    size_t size = 0;
    if (!fn || fn(&base, &size, reinterpret_cast<unsigned long long>(dev_ptr)) != 0) {
      set_error("cuMemGetAddressRange failed for %p", dev_ptr);
      return L4_ERR_CUDA;
    }
    off = (int64_t)(reinterpret_cast<unsigned long long>(dev_ptr) - base);
  }
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr));
  if (e != cudaSuccess) {
    set_error("cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  static_assert(sizeof(h) == L4_IPC_HANDLE_BYTES, "IPC handle is 64 bytes");
  std::memcpy(handle_out, &h, sizeof(h));
  if (offset_out) *offset_out = off;
  return L4_OK;
}

extern "C" l4_status l4_ipc_open_handle(const void* handle, void** dev_ptr_out) {
  L4_CHECK_ARG(handle && dev_ptr_out, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  void* p = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) {
    set_error("cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  *dev_ptr_out = p;
  return L4_OK;
}

extern "C" l4_status l4_ipc_close_handle(void* dev_ptr) {
  L4_CHECK_ARG(dev_ptr, "NULL argument");
  cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
  if (e != cudaSuccess) {
    set_error("cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  return L4_OK;
}

extern "C" l4_status l4_enable_peer_access(int32_t peer_device) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess && peer_device == dev) return L4_OK;
  int can = 0;
  if (e == cudaSuccess) e = cudaDeviceCanAccessPeer(&can, dev, peer_device);
  if (e == cudaSuccess && !can) {
    set_error("device %d cannot access peer %d", dev, peer_device);
    return L4_ERR_UNSUPPORTED;
  }
  if (e == cudaSuccess) {
    e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
      cudaGetLastError();
      e = cudaSuccess;
    }
  }
  if (e != cudaSuccess) {
    set_error("enable peer access: %s", cudaGetErrorString(e));
    cudaGetLastError();
    return L4_ERR_CUDA;
  }
  return L4_OK;
}
