/* Plain-C client of the l4 C ABI on a GPU (no Python in the loop): device calls through
 * include/l4.h with memory from the CUDA runtime.
 *  1. l4_decode_attention on BASELINE configs[0] (C1) with inputs drawn by the counter-based
 *     generator of synth/lcg.py (re-implemented below), checked against the FP64 oracle's values
 *     stored in tests/golden/c1_decode.txt (written by tests/golden/make_c1_decode_golden.py);
 *     tolerance 2e-3 (north star).
 *  2. l4_migrate of three pages between two device pools: destination ids are the pool's lowest
 *     free ids, the copied bytes equal the source bytes, the pool reports NO_PAGES when full.
 * Usage: abi_gpu <path to c1_decode.txt>; prints "ABI_GPU_OK" on success. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "l4.h"

#define CHECK(cond, msg)                                                        \
  do {                                                                          \
    if (!(cond)) {                                                              \
      fprintf(stderr, "FAIL %s (l4: %s)\n", msg, l4_last_error());             \
      return 1;                                                                 \
    }                                                                           \
  } while (0)
#define CUDA(x) CHECK((x) == cudaSuccess, #x)

static uint16_t bf16_bits(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return (uint16_t)(u >> 16); /* exact: the generator's values have 7 significant bits */
}

/* synth/lcg.py: x <- A x + C mod 2^64; value = (((x >> 33) mod 255) - 127) / 64 */
static void lcg_values(uint64_t seed, size_t n, uint16_t* out) {
  uint64_t x = seed;
  for (size_t i = 0; i < n; ++i) {
    x = 6364136223846793005ULL * x + 1442695040888963407ULL;
    out[i] = bf16_bits((float)((int)((x >> 33) % 255) - 127) / 64.0f);
  }
}

int main(int argc, char** argv) {
  CHECK(argc == 2, "usage: abi_gpu golden.txt");
  /* ---- C1 problem (synth/lcg.py c1_problem) */
  const int B = 4, Hq = 8, Hkv = 2, D = 128;
  const int32_t lens[4] = {16, 64, 256, 1024};
  int32_t indptr[5] = {0};
  for (int b = 0; b < B; ++b) indptr[b + 1] = indptr[b] + (lens[b] + 15) / 16;
  const int total = indptr[B], num_pages = total + 3;
  int32_t* indices = (int32_t*)malloc(sizeof(int32_t) * total);
  for (int i = 0; i < total; ++i) indices[i] = (31 * i + 7) % num_pages;
  const size_t nq = (size_t)B * Hq * D, nkv = (size_t)num_pages * Hkv * 16 * D;
  uint16_t *hq = malloc(2 * nq), *hk = malloc(2 * nkv), *hv = malloc(2 * nkv);
  lcg_values(1, nq, hq);
  lcg_values(2, nkv, hk);
  lcg_values(3, nkv, hv);

  void *dq, *dk, *dv, *dout, *dws;
  int32_t *dptr, *didx, *dlen;
  float* dlse;
  CUDA(cudaMalloc(&dq, 2 * nq));
  CUDA(cudaMalloc(&dk, 2 * nkv));
  CUDA(cudaMalloc(&dv, 2 * nkv));
  CUDA(cudaMalloc((void**)&dptr, sizeof(indptr)));
  CUDA(cudaMalloc((void**)&didx, sizeof(int32_t) * total));
  CUDA(cudaMalloc((void**)&dlen, sizeof(lens)));
  CUDA(cudaMalloc(&dout, sizeof(float) * nq));
  CUDA(cudaMalloc((void**)&dlse, sizeof(float) * B * Hq));
  CUDA(cudaMemcpy(dq, hq, 2 * nq, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dk, hk, 2 * nkv, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dv, hv, 2 * nkv, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dptr, indptr, sizeof(indptr), cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(didx, indices, sizeof(int32_t) * total, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(dlen, lens, sizeof(lens), cudaMemcpyHostToDevice));

  l4_decode_params p;
  memset(&p, 0, sizeof(p));
  p.batch = B;
  p.num_q_heads = Hq;
  p.num_kv_heads = Hkv;
  p.head_dim = D;
  p.page_size = 16;
  const size_t wsb = l4_decode_workspace_size(&p, total);
  CHECK(wsb > 0, "workspace_size");
  CUDA(cudaMalloc(&dws, wsb));
  CHECK(l4_decode_workspace_init(&p, dws, wsb, NULL) == L4_OK, "workspace_init");
  CHECK(l4_decode_attention(&p, dq, dk, dv, num_pages, dptr, didx, total, dlen, dout, dlse, dws, wsb, NULL) == L4_OK,
        "l4_decode_attention");
  CUDA(cudaDeviceSynchronize());
  float* out = malloc(sizeof(float) * nq);
  float lse[32];
  CUDA(cudaMemcpy(out, dout, sizeof(float) * nq, cudaMemcpyDeviceToHost));
  CUDA(cudaMemcpy(lse, dlse, sizeof(lse), cudaMemcpyDeviceToHost));

  FILE* f = fopen(argv[1], "r");
  CHECK(f != NULL, "open golden");
  double err = 0.0, lerr = 0.0;
  for (int i = 0; i < B * Hq; ++i) {
    int b, h;
    double g;
    CHECK(fscanf(f, "%d %d %lf", &b, &h, &g) == 3, "golden lse line");
    lerr = fmax(lerr, fabs((double)lse[b * Hq + h] - g));
  }
  for (size_t i = 0; i < nq; ++i) {
    double g;
    CHECK(fscanf(f, "%lf", &g) == 1, "golden out line");
    err = fmax(err, fabs((double)out[i] - g));
  }
  fclose(f);
  printf("l4_decode_attention C1 vs oracle golden: max abs err out %.3e lse %.3e\n", err, lerr);
  CHECK(err <= 2e-3 && lerr <= 2e-3, "decode parity");

  /* ---- l4_migrate: 3 pages of a 2-layer cache into a pool whose ids 0, 1 are taken */
  const int L = 2, P = 10;
  const size_t page_elems = (size_t)Hkv * 16 * D, pool_elems = (size_t)L * P * page_elems;
  uint16_t *hsk = malloc(2 * pool_elems), *hsv = malloc(2 * pool_elems), *back = malloc(2 * pool_elems);
  lcg_values(11, pool_elems, hsk);
  lcg_values(12, pool_elems, hsv);
  void *sk, *sv, *tk, *tv;
  CUDA(cudaMalloc(&sk, 2 * pool_elems));
  CUDA(cudaMalloc(&sv, 2 * pool_elems));
  CUDA(cudaMalloc(&tk, 2 * pool_elems));
  CUDA(cudaMalloc(&tv, 2 * pool_elems));
  CUDA(cudaMemcpy(sk, hsk, 2 * pool_elems, cudaMemcpyHostToDevice));
  CUDA(cudaMemcpy(sv, hsv, 2 * pool_elems, cudaMemcpyHostToDevice));
  CUDA(cudaMemset(tk, 0, 2 * pool_elems));
  CUDA(cudaMemset(tv, 0, 2 * pool_elems));
  l4_kv_view src = {0, sk, sv, P, L, (int64_t)(P * page_elems * 2), (int64_t)(page_elems * 2)};
  l4_kv_view dst = {0, tk, tv, P, L, (int64_t)(P * page_elems * 2), (int64_t)(page_elems * 2)};
  l4_page_pool* pool = NULL;
  CHECK(l4_pool_create(P, &pool) == L4_OK, "pool_create");
  int32_t taken[2];
  CHECK(l4_pool_alloc(pool, 2, taken) == L4_OK, "pool_alloc");
  const int32_t sp[3] = {7, 2, 5};
  int32_t dp[3] = {-1, -1, -1};
  CHECK(l4_migrate(&src, sp, 3, &dst, pool, dp, NULL, NULL) == L4_OK, "l4_migrate");
  CHECK(dp[0] == 2 && dp[1] == 3 && dp[2] == 4, "migrate: lowest free destination ids");
  CUDA(cudaDeviceSynchronize());
  for (int which = 0; which < 2; ++which) {
    CUDA(cudaMemcpy(back, which ? tv : tk, 2 * pool_elems, cudaMemcpyDeviceToHost));
    const uint16_t* s = which ? hsv : hsk;
    for (int l = 0; l < L; ++l)
      for (int i = 0; i < 3; ++i)
        CHECK(memcmp(back + ((size_t)l * P + dp[i]) * page_elems, s + ((size_t)l * P + sp[i]) * page_elems,
                     2 * page_elems) == 0, "migrate: bytes");
  }
  int32_t more[8];
  CHECK(l4_migrate(&src, sp, 3, &dst, pool, more, NULL, NULL) == L4_OK, "l4_migrate 2");
  CHECK(l4_migrate(&src, sp, 3, &dst, pool, more, NULL, NULL) == L4_ERR_NO_PAGES, "migrate: NO_PAGES when full");
  CHECK(l4_pool_num_free(pool) == 2, "migrate: pool unchanged after NO_PAGES");
  l4_pool_destroy(pool);
  printf("ABI_GPU_OK\n");
  return 0;
}
