/* Plain-C use of the C-ABI (include/rqa_b200.h): one analysis through rqa_run.
 * Build: gcc -O2 -o capi_example scripts/capi_example.c -Lpaper_2402_16853_b200 -lrqa_b200 \
 *          -Wl,-rpath,'$ORIGIN/../paper_2402_16853_b200'
 * Under `ncu --nvtx` the kernels carry the library's NVTX ranges
 * (rqa_run_prec > rqa.launch_rows), profiles/r02_nvtx_ncu.txt. */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "../include/rqa_b200.h"

int main(void) {
  const int n = 3000;
  double* s = malloc(n * sizeof(double));
  for (int i = 0; i < n; ++i) s[i] = (double)((i * 7919) % 1000) / 1000.0;
  int64_t *d = calloc(n + 1, 8), *v = calloc(n + 1, 8), *w = calloc(n + 1, 8), p = 0;
  double tim[RQA_TIMING_SLOTS];
  char err[256];
  /* m = 2, tau = 1, L2 (metric 1), radius 0.1, main diagonal kept, device 0 */
  const int rc = rqa_run(s, n, 2, 1, 1, 0.1, 0, 0, d, v, w, &p, tim, err, sizeof err);
  if (rc != 0) {
    fprintf(stderr, "rqa_run failed (%d): %s\n", rc, err);
    return 1;
  }
  printf("recurrence points %lld, kernel %.3f ms\n", (long long)p, tim[1] * 1e3);
  free(s); free(d); free(v); free(w);
  return 0;
}
