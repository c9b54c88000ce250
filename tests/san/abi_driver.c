/* ASan/UBSan driver for libcorr.so's host-side C ABI (test infrastructure).  Linked
 * against a libcorr build whose api.cu host code is compiled with -fsanitize=address,undefined
 * (tests/test_sanitizers.py).  Exercises argument validation and error reporting -- every call
 * here returns before any device work -- and, when no CUDA device is present, the "no CUDA device
 * -> CORR_E_CUDA" paths.  Exit 0 = every status as documented in include/corr.h, sanitizers clean. */
#include <stdio.h>
#include <string.h>

#include "corr.h"

static int fails = 0;
#define EXPECT(call, code)                                                                 \
  do {                                                                                     \
    int rc_ = (call);                                                                      \
    if (rc_ != (code)) {                                                                   \
      fprintf(stderr, "%s: got %d want %d (%s)\n", #call, rc_, (code), corr_last_error()); \
      ++fails;                                                                             \
    }                                                                                      \
  } while (0)

int main(int argc, char** argv) {
  const int no_device = argc > 1 && strcmp(argv[1], "--no-device") == 0;
  float v[64];
  for (int i = 0; i < 64; ++i) v[i] = (float)i;
  corr_field* f = NULL;
  corr_box bx = {0, 0, 0, 1, 1, 1};
  int64_t idx[2] = {0, 1}, cnt = 0;
  float out[2];
  int32_t d = 0;
  EXPECT(corr_field_create(v, 4, 4, 1, 4, 0, NULL, NULL), CORR_E_INVAL);   /* out NULL */
  EXPECT(corr_field_create(NULL, 4, 4, 1, 4, 0, NULL, &f), CORR_E_INVAL);  /* values NULL */
  EXPECT(corr_field_create(v, 0, 4, 1, 4, 0, NULL, &f), CORR_E_INVAL);     /* dims < 1 */
  EXPECT(corr_field_create(v, 4, 4, 1, 1, 0, NULL, &f), CORR_E_INVAL);     /* members < 2 */
  EXPECT(corr_field_create(v, 4, 4, 1, 5000, 0, NULL, &f), CORR_E_INVAL);  /* members > 4096 */
  if (no_device) EXPECT(corr_field_create(v, 4, 4, 1, 4, 0, NULL, &f), CORR_E_CUDA);
  EXPECT(corr_field_update(NULL, v, NULL), CORR_E_INVAL);
  EXPECT(corr_field_destroy(NULL), CORR_OK);
  EXPECT(corr_field_info(NULL, &d, &d, &d, &d, &d), CORR_E_INVAL);
  EXPECT(corr_field_aggregate(NULL, 2, 2, 2, NULL, &f), CORR_E_INVAL);
  EXPECT(corr_eval_pairs(NULL, NULL, CORR_KSG, 3, idx, idx, 2, out, NULL), CORR_E_INVAL);
  EXPECT(corr_region_max(NULL, NULL, CORR_KSG, 3, &bx, &bx, 1, 10, 1, out, idx, NULL), CORR_E_INVAL);
  EXPECT(corr_ksg_debug(NULL, NULL, 3, idx, idx, 2, out, NULL, NULL, NULL), CORR_E_INVAL);
  EXPECT(corr_check(NULL, NULL), CORR_E_INVAL);
  EXPECT(corr_ksg_comparisons(0, NULL, 0), CORR_E_INVAL);
  EXPECT(corr_ksg_nan_pairs(0, NULL, 0), CORR_E_INVAL);
  EXPECT(corr_gemm_flops(0, NULL, NULL, 0), CORR_E_INVAL);
  if (no_device) {
    EXPECT(corr_ksg_comparisons(0, &cnt, 1), CORR_E_CUDA);
    EXPECT(corr_ksg_nan_pairs(0, &cnt, 1), CORR_E_CUDA);
  }
  if (corr_launch_count() != 0) ++fails;
  if (fails) return 1;
  printf("ok\n");
  return 0;
}
