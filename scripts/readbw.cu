// Read-bandwidth probe (development evidence only, not product code): how fast can a
// B200 stream bytes from HBM into the SMs?  Two readers over one large buffer:
//   ldg : 128-bit ld.global.nc (L1 no-allocate), 8 loads in flight per thread, grid-stride
//   tma : cp.async.bulk 1-D copies of 8 KB into a per-CTA smem ring (what decode_kernel does)
// Built by scripts/build_readbw.sh into scripts/readbw.so, driven by scripts/readbw.py.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__global__ void ldg_kernel(const uint4* __restrict__ p, size_t n16, unsigned long long* sink) {
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  size_t i = tid;
  for (; i + 7 * stride < n16; i += 8 * stride) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(p + i + u * stride));
#pragma unroll
    for (int u = 0; u < 8; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) {
    const uint4 v = p[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int kStages, int kChunk>
__global__ void tma_kernel(const char* __restrict__ p, size_t nbytes, unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kStages];
  const uint32_t sb = smem_u32(smem);
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t nchunks = nbytes / kChunk;
  uint32_t k = 0;
  uint32_t acc = 0;
  auto wait = [&](uint32_t q) {
    const uint32_t bar = smem_u32(&full[q % kStages]);
    const uint32_t par = (q / kStages) & 1;
    asm volatile(
        "{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra D;\n\tbra W;\nD:\n\t}" ::"r"(bar),
        "r"(par)
        : "memory");
    acc ^= *reinterpret_cast<volatile uint32_t*>(smem + (q % kStages) * kChunk);
  };
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++k) {
    if (k >= kStages) wait(k - kStages);
    const uint32_t st = k % kStages;
    const uint32_t bar = smem_u32(&full[st]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(kChunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     sb + st * kChunk),
                 "l"(p + c * kChunk), "r"(kChunk), "r"(bar)
                 : "memory");
  }
  for (uint32_t q = k > kStages ? k - kStages : 0; q < k; ++q) wait(q);
  if (acc == 0x12345678u) atomicAdd(sink, 1ull);
}

}  // namespace

extern "C" int probe_ldg(const void* p, size_t nbytes, int grid, int block, void* sink, void* stream) {
  ldg_kernel<<<grid, block, 0, (cudaStream_t)stream>>>((const uint4*)p, nbytes / 16, (unsigned long long*)sink);
  return (int)cudaGetLastError();
}

extern "C" int probe_tma(const void* p, size_t nbytes, int grid, int stages_kb, void* sink, void* stream) {
  // stages_kb selects the ring: 64 (8 x 8 KB) or 128 (16 x 8 KB) or 96 (12 x 8 KB)
  cudaStream_t st = (cudaStream_t)stream;
  if (stages_kb == 64) {
    cudaFuncSetAttribute(tma_kernel<8, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192);
    tma_kernel<8, 8192><<<grid, 32, 8 * 8192, st>>>((const char*)p, nbytes, (unsigned long long*)sink);
  } else if (stages_kb == 96) {
    cudaFuncSetAttribute(tma_kernel<12, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 12 * 8192);
    tma_kernel<12, 8192><<<grid, 32, 12 * 8192, st>>>((const char*)p, nbytes, (unsigned long long*)sink);
  } else {
    cudaFuncSetAttribute(tma_kernel<16, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * 8192);
    tma_kernel<16, 8192><<<grid, 32, 16 * 8192, st>>>((const char*)p, nbytes, (unsigned long long*)sink);
  }
  return (int)cudaGetLastError();
}
