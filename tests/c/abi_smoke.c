/* Plain-C client of the l4 C ABI (include/l4.h): proves the boundary is usable without Python.
 * Host-only calls (partition, refinement, QoE fit, page pool) run anywhere; the device calls are
 * expected to return L4_ERR_CUDA on a host without a B200 and L4_OK with one. */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "l4.h"

#define CHECK(cond, msg)                                      \
  do {                                                        \
    if (!(cond)) {                                            \
      fprintf(stderr, "FAIL %s: %s\n", msg, l4_last_error()); \
      return 1;                                               \
    }                                                         \
  } while (0)

int main(void) {
  /* SURVEY A.2 hand example: (I,O) = (2,1),(3,3),(10,4), D = (0,0,0,0,1), 1 B/token at 1 B/s */
  const int64_t I[3] = {2, 3, 10}, O[3] = {1, 3, 4};
  l4_partition_params pp;
  memset(&pp, 0, sizeof(pp));
  pp.num_instances = 2;
  pp.migrate_bandwidth_Bps = 1.0;
  pp.kv_bytes_per_token = 1;
  pp.qoe_d[4] = 1.0;
  pp.stage_cost_mode = 1;
  l4_stage st[4];
  int32_t ns = 0;
  double obj = 0;
  CHECK(l4_partition(&pp, I, O, 3, st, &ns, &obj) == L4_OK, "partition");
  CHECK(obj == 32.0 && ns == 2 && st[0].hi == 8 && st[1].lo == 8, "partition value");
  pp.num_instances = 0;
  CHECK(l4_partition(&pp, I, O, 3, st, &ns, &obj) == L4_ERR_INVALID_ARG, "partition E=0");

  l4_page_pool* pool = NULL;
  int32_t pages[4];
  CHECK(l4_pool_create(5, &pool) == L4_OK, "pool_create");
  CHECK(l4_pool_alloc(pool, 3, pages) == L4_OK && pages[0] == 0 && pages[2] == 2, "pool_alloc");
  CHECK(l4_pool_alloc(pool, 3, pages) == L4_ERR_NO_PAGES && l4_pool_num_free(pool) == 2, "pool no pages");
  l4_pool_destroy(pool);

  l4_refine_params rp;
  memset(&rp, 0, sizeof(rp));
  rp.qoe_d[4] = 1.0;
  rp.ema_alpha = 1.0;
  rp.min_traffic = 1;
  rp.lo = 0;
  rp.hi = 1000000;
  const int64_t lI[2] = {1, 1}, lL[2] = {100, 200}, sp[2] = {0, 2}, sI[2] = {1, 1}, sL[2] = {300, 400};
  double nb = 0;
  int64_t raw = 0, split = 0;
  CHECK(l4_refine_boundary(&rp, lI, lL, 2, 1, sp, sI, sL, 250.0, &nb, &raw, &split) == L4_OK, "refine");
  CHECK(nb == (double)raw && split >= 0, "refine value");

  double F[6 * 5], Q[6], D[5], rms;
  for (int i = 0; i < 6; ++i) {
    F[i * 5 + 0] = 1;
    F[i * 5 + 1] = i + 1;
    F[i * 5 + 2] = 10 * i + 3;
    F[i * 5 + 3] = (i + 2) * (i + 7);
    F[i * 5 + 4] = 100 + 37 * i * i;
    Q[i] = 0.5 + 0.25 * F[i * 5 + 1] + 1e-3 * F[i * 5 + 4];
  }
  CHECK(l4_qoe_fit(F, Q, 6, 0x13u, D, &rms) == L4_OK, "qoe_fit");
  CHECK(fabs(D[0] - 0.5) < 1e-9 && fabs(D[1] - 0.25) < 1e-9 && fabs(D[4] - 1e-3) < 1e-12, "qoe_fit value");

  l4_decode_params dp;
  memset(&dp, 0, sizeof(dp));
  dp.batch = 4;
  dp.num_q_heads = 8;
  dp.num_kv_heads = 2;
  dp.head_dim = 128;
  dp.page_size = 16;
  size_t ws = l4_decode_workspace_size(&dp, 85);
  printf("l4 %s: partition/pool/refine/qoe OK; decode workspace %zu bytes (%s)\n", l4_version(), ws,
         ws ? "device present" : l4_last_error());
  return 0;
}
