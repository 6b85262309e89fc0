/* Host cost per call of the C ABI (no Python): N back-to-back small
 * AllReduce calls of m virtual ranks on device 0, timed on the host.
 *   gcc -O2 -I include -I /usr/local/cuda/include scripts/c_overhead.c -L paper_1910_04940_b200 \
 *       -lblink -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,$PWD/paper_1910_04940_b200 -o /tmp/co */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <time.h>

#include "blink.h"

static double now_us(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

int main(void) {
  for (int m = 1; m <= 8; m *= 2) {
    blink_comm_t c[8];
    int devs[8] = {0};
    void *s[8], *r[8];
    blink_init_all(c, m, devs, NULL, NULL);
    for (int k = 0; k < m; ++k) {
      cudaMalloc(&s[k], 4096);
      cudaMalloc(&r[k], 4096);
    }
    const int N = 5000;
    for (int it = 0; it < 100; ++it)
      for (int k = 0; k < m; ++k) blink_allreduce(c[k], s[k], r[k], 256, BLINK_FLOAT32, BLINK_SUM, NULL);
    cudaDeviceSynchronize();
    double t0 = now_us();
    for (int it = 0; it < N; ++it)
      for (int k = 0; k < m; ++k) blink_allreduce(c[k], s[k], r[k], 256, BLINK_FLOAT32, BLINK_SUM, NULL);
    double t1 = now_us();
    cudaDeviceSynchronize();
    double t2 = now_us();
    printf("m=%d: host %.2f us per collective, wall %.2f us\n", m, (t1 - t0) / N, (t2 - t0) / N);
    for (int k = 0; k < m; ++k) blink_destroy(c[k]);
  }
  return 0;
}
