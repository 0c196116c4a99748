/* Plain-C consumer of include/mk_strassen.h: links libmk_strassen.so and exercises the
 * host-only entry points (no GPU needed). Built and run by tests/test_abi.py. */
#include <stdio.h>
#include <string.h>
#include "mk_strassen.h"

static int fails = 0;
#define CHECK(cond)                                             \
  do {                                                          \
    if (!(cond)) {                                              \
      printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
      ++fails;                                                  \
    }                                                           \
  } while (0)

int main(void) {
  int lv = -1;
  CHECK(mk_version() >= 2);
  /* BasePolicy.naive_cutoff(1024) at n = 8192: leaf when n <= 1024 -> 3 halvings */
  CHECK(mk_levels_for_policy(8192, 2, 1024, MK_ALGO_WINOGRAD_BLOCK, &lv) == MK_OK && lv == 3);
  CHECK(mk_levels_for_policy(16384, 2, 4096, MK_ALGO_STRASSEN, &lv) == MK_OK && lv == 2);
  CHECK(mk_levels_for_policy(1, 0, 1, MK_ALGO_IN_PLACE, &lv) == MK_OK && lv == 0);
  CHECK(mk_levels_for_policy(16, 9, 1, MK_ALGO_IN_PLACE, &lv) == MK_ERR_ARG);
  CHECK(strlen(mk_last_error()) > 0);
  /* workspace: in-place none; depth-first partial at L=1 two (n/2)^2 slots */
  CHECK(mk_workspace_bytes(MK_ALGO_IN_PLACE, 1024, 3) == 0);
  CHECK(mk_partial_workspace_bytes(MK_ALGO_WINOGRAD_BLOCK, 1024, 1) == (size_t)2 * 512 * 512 * 8);
  CHECK(mk_workspace_bytes(MK_ALGO_WINOGRAD_BLOCK, 1000, 1) == 0); /* not a power of two */
  CHECK(mk_product_count(MK_ALGO_WINOGRAD_BLOCK, 3) == 343);
  CHECK(mk_product_count(MK_ALGO_WINOGRAD_KNUTH_8CALL, 2) == 64);
  CHECK(mk_rect_workspace_bytes(MK_ALGO_STRASSEN, 300, 129, 517, 2) > 0);
  CHECK(mk_set_option(MK_OPT_FUSE_PREADDS, 0) == MK_OK);
  /* argument errors are reported before any CUDA call */
  CHECK(mk_strassen(MK_ALGO_WINOGRAD_BLOCK, 0, 6, 0, 6, 0, 6, 6, 1, 0, 0, 0) == MK_ERR_DIMENSION);
  CHECK(mk_strassen(99, 0, 8, 0, 8, 0, 8, 8, 1, 0, 0, 0) == MK_ERR_ARG);
  CHECK(mk_dgemm(0, 4, 0, 4, 0, 4, 0, 4, 4, 0) == MK_ERR_DIMENSION);
  if (fails == 0) printf("abi_check ok\n");
  return fails ? 1 : 0;
}
