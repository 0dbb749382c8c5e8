/* Plain C11 client of include/sttsv.h: the header compiles as C (not C++), links
 * against libsttsv.so, and the calls behave as documented.
 *
 *   abi_c11            host-only checks (status strings, validation errors that
 *                      are raised before any device work, edge sharding)
 *   abi_c11 gpu        also: plan_create / apply_host / destroy on the paper's
 *                      Fig. 1 hypergraph with w(e) = |e| and
 *                      x = 1, whose product is the degree vector:
 *                      (3,2,3,4,2,3,3,1).
 * Exit status 0 on success; prints the first failure. */
#include <math.h>
#include <stdio.h>
#include <string.h>

#include "sttsv.h"

#define CHECK(cond, ...)                          \
  do {                                            \
    if (!(cond)) {                                \
      fprintf(stderr, "FAIL %s:%d: ", __FILE__, __LINE__); \
      fprintf(stderr, __VA_ARGS__);               \
      fprintf(stderr, "\n");                      \
      return 1;                                   \
    }                                             \
  } while (0)

static int host_checks(void) {
  CHECK(strcmp(sttsv_status_string(STTSV_OK), "STTSV_OK") == 0, "status string");
  CHECK(strcmp(sttsv_status_string(STTSV_ERR_UNSORTED), "STTSV_ERR_UNSORTED") == 0, "status string");
  CHECK(strstr(sttsv_version(), "sm_100a") != NULL, "version %s", sttsv_version());
  sttsv_plan_t p = (sttsv_plan_t)0x1;
  const int32_t sizes[1] = {2};
  const int32_t unsorted[2] = {3, 1};
  sttsv_status_t st = sttsv_plan_create(&p, 10, 4, 1, sizes, unsorted, NULL, 0, 1, 0, NULL, 0);
  CHECK(st == STTSV_ERR_UNSORTED && p == NULL, "unsorted edge: %d", (int)st);
  CHECK(strlen(sttsv_last_error()) > 0, "last error text");
  const int32_t out_of_range[2] = {1, 10};
  st = sttsv_plan_create(&p, 10, 4, 1, sizes, out_of_range, NULL, 0, 1, 0, NULL, 0);
  CHECK(st == STTSV_ERR_VERTEX_RANGE, "vertex range: %d", (int)st);
  st = sttsv_plan_create(&p, 10, STTSV_MAX_RANK + 1, 1, sizes, unsorted, NULL, 0, 1, 0, NULL, 0);
  CHECK(st == STTSV_ERR_INVALID_ARGUMENT, "rank cap: %d", (int)st);
  CHECK(sttsv_destroy(NULL) == STTSV_OK, "destroy(NULL)");
  /* sharding: bucket slices of sizes {2,3,2,2,3} over 2 ranks */
  const int32_t sz[5] = {2, 3, 2, 2, 3};
  int64_t e0[5], e1[5], c0 = 0, c1 = 0;
  CHECK(sttsv_shard_edges(5, sz, 3, 2, 0, e0, &c0) == STTSV_OK, "shard 0");
  CHECK(sttsv_shard_edges(5, sz, 3, 2, 1, e1, &c1) == STTSV_OK, "shard 1");
  CHECK(c0 + c1 == 5, "shard counts %lld + %lld", (long long)c0, (long long)c1);
  return 0;
}

static int gpu_checks(void) {
  /* PAPER.md Fig. 1 (1-based): {2,3,4,7},{1,3,4,6},{1,2,3,8},{4,5,6,7},{1,4,6},{5,7} */
  const int32_t sizes[6] = {4, 4, 4, 4, 3, 2};
  const int32_t idx[21] = {1, 2, 3, 6, 0, 2, 3, 5, 0, 1, 2, 7, 3, 4, 5, 6, 0, 3, 5, 4, 6};
  const double expect[8] = {3, 2, 3, 4, 2, 3, 3, 1};
  double x[8], y[8];
  for (int i = 0; i < 8; ++i) x[i] = 1.0;
  sttsv_plan_t p = NULL;
  sttsv_status_t st = sttsv_plan_create(&p, 8, 4, 6, sizes, idx, NULL, 0, 1, 0, NULL, 0);
  CHECK(st == STTSV_OK && p != NULL, "plan_create: %s (%s)", sttsv_status_string(st), sttsv_last_error());
  st = sttsv_apply_host(p, x, y);
  CHECK(st == STTSV_OK, "apply_host: %s (%s)", sttsv_status_string(st), sttsv_last_error());
  for (int i = 0; i < 8; ++i) CHECK(fabs(y[i] - expect[i]) <= 1e-13, "y[%d] = %.17g, expected %g", i, y[i], expect[i]);
  sttsv_plan_info_t info;
  CHECK(sttsv_plan_info(p, &info) == STTSV_OK && info.n_active == 8 && info.incidences == 21, "plan_info");
  CHECK(sttsv_destroy(p) == STTSV_OK, "destroy");
  printf("fig1 y = (%g,%g,%g,%g,%g,%g,%g,%g)\n", y[0], y[1], y[2], y[3], y[4], y[5], y[6], y[7]);
  return 0;
}

int main(int argc, char** argv) {
  int rc = host_checks();
  if (rc) return rc;
  if (argc > 1 && strcmp(argv[1], "gpu") == 0) rc = gpu_checks();
  if (!rc) printf("abi_c11 ok\n");
  return rc;
}
