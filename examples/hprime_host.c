/*
 * Plain-C client of the C ABI (include/lfbp_hprime.h): what a non-Python
 * host would write.  Builds H for a small odd shape, runs the host-to-host
 * H -> H' path (lfbp_hprime_host), then the inverse, and checks that the
 * round trip returns H bit for bit (the map is an involution for odd
 * n_s, n_t; reference test_transform.py:157-162) and that the single-element
 * known answer of test_transform.py:108-115 holds.
 *
 *   gcc -std=c99 -O2 -Iinclude examples/hprime_host.c \
 *       -Lpaper_2003_09133_b200 -lhprime -Wl,-rpath,$PWD/paper_2003_09133_b200 -o hprime_host
 *   ./hprime_host          (needs a GPU)
 *   ./hprime_host --abi    (no GPU: dims checks and version only)
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lfbp_hprime.h"

static int check(int rc, const char* what) {
  if (rc != LFBP_OK) fprintf(stderr, "%s failed: status %d: %s\n", what, rc, lfbp_last_error());
  return rc;
}

int main(int argc, char** argv) {
  const int64_t dims[5] = {21, 19, 7, 5, 3};
  const int64_t bad[5] = {21, 19, 6, 5, 3}; /* even n_x: InvalidDims */
  const int64_t even[5] = {4, 5, 3, 3, 1};  /* 45 dropped elements */
  printf("%s\n", lfbp_version());
  if (lfbp_check_dims(dims) != LFBP_OK || lfbp_check_dims(bad) != LFBP_ERR_INVALID_DIMS) return 1;
  if (lfbp_dropped_source_count(even) != 45 || lfbp_dropped_source_count(dims) != 0) return 1;
  if (argc > 1 && strcmp(argv[1], "--abi") == 0) {
    printf("abi ok\n");
    return 0;
  }
  const size_t n = (size_t)(dims[0] * dims[1] * dims[2] * dims[3] * dims[4]);
  float* h = malloc(n * sizeof(float));
  float* hp = malloc(n * sizeof(float));
  float* back = malloc(n * sizeof(float));
  if (!h || !hp || !back) return 1;
  uint32_t x = 12345u; /* xorshift: arbitrary bit patterns, NaN payloads included */
  for (size_t i = 0; i < n; ++i) {
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    memcpy(&h[i], &x, 4);
  }
  if (check(lfbp_hprime_host(h, hp, dims, LFBP_F32, 0, 0, LFBP_HOST_REGISTER), "forward")) return 1;
  if (check(lfbp_hprime_host(hp, back, dims, LFBP_F32, 1, 0, LFBP_HOST_REGISTER), "inverse")) return 1;
  if (memcmp(h, back, n * sizeof(float)) != 0) {
    fprintf(stderr, "round trip differs\n");
    return 1;
  }
  /* single element (5,5,3,3,1): H[0,0,2,2,0] = 1 -> H'[4,4,0,0,0] = 1, nothing else */
  const int64_t d1[5] = {5, 5, 3, 3, 1};
  double one[225] = {0}, out[225];
  one[0 + 5 * (0 + 5 * (2 + 3 * 2))] = 1.0;
  if (check(lfbp_hprime_host(one, out, d1, LFBP_F64, 0, 0, 0), "single element")) return 1;
  for (int i = 0; i < 225; ++i) {
    const double want = (i == 4 + 5 * 4) ? 1.0 : 0.0;
    if (out[i] != want) {
      fprintf(stderr, "single element: H'[%d] = %g\n", i, out[i]);
      return 1;
    }
  }
  printf("round trip and single-element KAT ok (%zu elements)\n", n);
  free(h);
  free(hp);
  free(back);
  return 0;
}
