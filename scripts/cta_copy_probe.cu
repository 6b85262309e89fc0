// Per-CTA copy throughput on one B200: how fast can ONE CTA move a
// contiguous HBM region, and what does the rate depend on?  (The tree
// executor's deep-tree channels run with few CTAs each; the pipeline fit in
// profiles/pipeline_r02.json puts one channel CTA at ~44 GB/s.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cta_copy_probe scripts/cta_copy_probe.cu
//   /tmp/cta_copy_probe
//
// Variants, each a grid of G CTAs copying G disjoint 8 MiB regions:
//   tma   : one thread issues cp.async.bulk loads into an S-stage ring of T-byte
//           tiles (mbarrier complete_tx), another thread issues the bulk stores
//           (bulk_group; a stage is reused after wait_group.read) -- the
//           executor's copy pattern;
//   lsu   : every thread copies 16-byte vectors with U loads in flight.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t phase) {
  asm volatile(
      "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(smem_u32(b)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_store(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

template <int D>
__device__ __forceinline__ void wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(D) : "memory");
}

// S stages of T bytes; store depth D (groups kept in flight before a stage is released)
template <int D>
__global__ void tma_copy(char* dst, const char* src, int64_t per_cta, int T, int S) {
  extern __shared__ __align__(128) char ring[];
  __shared__ uint64_t full[16], empty[16];
  const int64_t base = int64_t(blockIdx.x) * per_cta;
  const int ntiles = int(per_cta / T);
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // producer
    for (int g = 0; g < ntiles; ++g) {
      const int s = g % S;
      if (g >= S) mbar_wait(&empty[s], ((g / S) - 1) & 1);
      mbar_expect_tx(&full[s], T);
      tma_load(ring + size_t(s) * T, src + base + int64_t(g) * T, T, &full[s]);
    }
  } else if (threadIdx.x == 32) {  // store
    int kept = 0;
    for (int g = 0; g < ntiles; ++g) {
      const int s = g % S;
      mbar_wait(&full[s], (g / S) & 1);
      tma_store(dst + base + int64_t(g) * T, ring + size_t(s) * T, T);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++kept > D) {
        wait_read<D>();
        const int r = (g - D) % S;
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[r])) : "memory");
        --kept;
      }
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
  __syncthreads();
}

template <int U>
__global__ void lsu_copy(char* dst, const char* src, int64_t per_cta) {
  const uint4* s = reinterpret_cast<const uint4*>(src + int64_t(blockIdx.x) * per_cta);
  uint4* d = reinterpret_cast<uint4*>(dst + int64_t(blockIdx.x) * per_cta);
  const int64_t n = per_cta / 16;
  for (int64_t i = threadIdx.x; i < n; i += int64_t(blockDim.x) * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + int64_t(u) * blockDim.x;
      if (j < n) v[u] = __ldcg(s + j);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t j = i + int64_t(u) * blockDim.x;
      if (j < n) __stcg(d + j, v[u]);
    }
  }
}

int main() {
  const int64_t per_cta = 8 << 20;
  const int Gmax = 148;
  char *a, *b;
  cudaMalloc(&a, per_cta * Gmax);
  cudaMalloc(&b, per_cta * Gmax);
  cudaMemset(a, 1, per_cta * Gmax);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaFuncSetAttribute(tma_copy<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 << 10);
  cudaFuncSetAttribute(tma_copy<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 << 10);
  cudaFuncSetAttribute(tma_copy<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 << 10);
  auto run = [&](const char* name, int G, auto launch) {
    launch(G);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch(G);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= 5;
    const double gbs = double(per_cta) * G / (ms * 1e-3) / 1e9;
    printf("%-26s G=%3d  %8.1f GB/s total  %6.1f GB/s per CTA (copy bytes)\n", name, G, gbs, gbs / G);
    fflush(stdout);
  };
  for (int G : {1, 8, 148}) {
    for (int T : {16384, 32768, 65536}) {
      for (int S : {3, 4, 6}) {      // S > D (a stage is released D groups after its store)
        if (size_t(T) * S > (200 << 10)) continue;
        char nm[64];
        snprintf(nm, sizeof nm, "tma T=%dK S=%d D=2", T >> 10, S);
        run(nm, G, [&](int g) { tma_copy<2><<<g, 64, size_t(T) * S>>>(b, a, per_cta, T, S); });
      }
    }
    run("tma T=32K S=6 D=4", G, [&](int g) { tma_copy<4><<<g, 64, 32768 * 6>>>(b, a, per_cta, 32768, 6); });
    run("tma T=32K S=6 D=1", G, [&](int g) { tma_copy<1><<<g, 64, 32768 * 6>>>(b, a, per_cta, 32768, 6); });
    run("lsu U=4 256 thr", G, [&](int g) { lsu_copy<4><<<g, 256>>>(b, a, per_cta); });
    run("lsu U=8 512 thr", G, [&](int g) { lsu_copy<8><<<g, 512>>>(b, a, per_cta); });
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
  return 0;
}
