/* Plain C use of the C ABI (include/blink.h): no Python, no torch.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/allreduce_c.c \
 *       -L paper_1910_04940_b200 -lblink -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1910_04940_b200 -o /tmp/allreduce_c && /tmp/allreduce_c [m] [count]
 *
 * m virtual ranks on device 0 (blink_init_all with a repeated device, the
 * single-process mode), then on the emulated DGX-1V link graph: an int32
 * SUM AllReduce (exact under any tree, so the expected value is a closed
 * form: sum_r (r * 1000 + i) = 1000 m(m-1)/2 + m i), AVG (500 (m-1) + i), a
 * Broadcast from the last rank, and the error path of a bad root.  Prints
 * "c api ok".
 */
#include <cuda_runtime_api.h>
#include <stdio.h>
#include <stdlib.h>

#include "blink.h"

#define CK(x)                                                                 \
  do {                                                                        \
    blink_result_t r_ = (x);                                                  \
    if (r_ != BLINK_SUCCESS) {                                                \
      fprintf(stderr, "%s:%d %s: %s (%s)\n", __FILE__, __LINE__, #x,          \
              blink_result_string(r_), blink_last_error(NULL));               \
      exit(1);                                                                \
    }                                                                         \
  } while (0)
#define CU(x)                                                                 \
  do {                                                                        \
    cudaError_t e_ = (x);                                                     \
    if (e_ != cudaSuccess) {                                                  \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      exit(1);                                                                \
    }                                                                         \
  } while (0)

/* App. B DGX-1V hybrid cube-mesh (pairs with 2 NVLinks get capacity 2). */
static const int kPairs[][3] = {{0, 1, 1}, {0, 2, 1}, {0, 3, 2}, {0, 4, 2}, {1, 2, 2}, {1, 3, 1},
                                {1, 5, 2}, {2, 3, 2}, {2, 6, 1}, {3, 7, 1}, {4, 5, 1}, {4, 6, 1},
                                {4, 7, 2}, {5, 6, 2}, {5, 7, 1}, {6, 7, 2}};

static int run(int m, size_t count, const blink_graph_t* graph, const char* what) {
  blink_comm_t comms[16];
  int devs[16] = {0};
  void* send[16];
  void* recv[16];
  int* host = (int*)malloc(count * sizeof(int));
  CK(blink_init_all(comms, m, devs, graph, NULL));
  for (int r = 0; r < m; ++r) {
    for (size_t i = 0; i < count; ++i) host[i] = r * 1000 + (int)i;
    CU(cudaMalloc(&send[r], count * sizeof(int)));
    CU(cudaMalloc(&recv[r], count * sizeof(int)));
    CU(cudaMemcpy(send[r], host, count * sizeof(int), cudaMemcpyHostToDevice));
  }
  /* every rank calls; the single-process comm launches once all have */
  for (int r = 0; r < m; ++r)
    CK(blink_allreduce(comms[r], send[r], recv[r], count, BLINK_INT32, BLINK_SUM, NULL));
  CU(cudaDeviceSynchronize());
  for (int r = 0; r < m; ++r) {
    CU(cudaMemcpy(host, recv[r], count * sizeof(int), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < count; ++i) {
      const int want = 1000 * m * (m - 1) / 2 + m * (int)i;
      if (host[i] != want) {
        fprintf(stderr, "%s: allreduce rank %d [%zu] = %d, want %d\n", what, r, i, host[i], want);
        return 1;
      }
    }
  }
  /* AVG (R#28): the same sum divided by m at the tree root = 500 (m-1) + i */
  for (int r = 0; r < m; ++r)
    CK(blink_allreduce(comms[r], send[r], recv[r], count, BLINK_INT32, BLINK_AVG, NULL));
  CU(cudaDeviceSynchronize());
  for (int r = 0; r < m; ++r) {
    CU(cudaMemcpy(host, recv[r], count * sizeof(int), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < count; ++i)
      if (host[i] != 500 * (m - 1) + (int)i) {
        fprintf(stderr, "%s: avg rank %d [%zu] = %d\n", what, r, i, host[i]);
        return 1;
      }
  }
  for (int r = 0; r < m; ++r)
    CK(blink_broadcast(comms[r], r == m - 1 ? send[r] : NULL, recv[r], count, BLINK_INT32, m - 1, NULL));
  CU(cudaDeviceSynchronize());
  for (int r = 0; r < m; ++r) {
    CU(cudaMemcpy(host, recv[r], count * sizeof(int), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < count; ++i)
      if (host[i] != (m - 1) * 1000 + (int)i) {
        fprintf(stderr, "%s: broadcast rank %d [%zu] = %d\n", what, r, i, host[i]);
        return 1;
      }
  }
  if (blink_broadcast(comms[0], send[0], recv[0], count, BLINK_INT32, m, NULL) !=
      BLINK_ERR_INVALID_ARGUMENT) {
    fprintf(stderr, "%s: bad root accepted\n", what);
    return 1;
  }
  blink_stats_t st;
  CK(blink_get_stats(comms[0], &st));
  printf("%s: m=%d count=%zu ok (%d launches)\n", what, m, count, (int)st.launches);
  for (int r = 0; r < m; ++r) {
    CU(cudaFree(send[r]));
    CU(cudaFree(recv[r]));
    CK(blink_destroy(comms[r]));
  }
  free(host);
  return 0;
}

int main(int argc, char** argv) {
  const int m = argc > 1 ? atoi(argv[1]) : 8;
  const size_t count = argc > 2 ? (size_t)atoll(argv[2]) : 1000003;
  if (run(m, count, NULL, "switch") != 0) return 1;
  blink_link_t links[32];
  blink_node_kind_t kinds[8];
  for (int v = 0; v < 8; ++v) kinds[v] = BLINK_NODE_GPU;
  const int np = (int)(sizeof kPairs / sizeof kPairs[0]);
  for (int k = 0; k < np; ++k) {
    links[k].src = kPairs[k][0];
    links[k].dst = kPairs[k][1];
    links[k].capacity = kPairs[k][2];
    links[k].bidirectional = 1;
  }
  blink_graph_t g = {8, kinds, np, links};
  if (run(8, count, &g, "dgx1v") != 0) return 1;
  if (run(8, 1001, &g, "dgx1v-small") != 0) return 1;
  printf("c api ok\n");
  return 0;
}
