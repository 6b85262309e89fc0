// PDL probe: per-call device time of back-to-back launches in the executor's
// shape (148 CTAs x 256 threads, 200 KB dynamic smem, a streaming copy of
// `bytes`, last-CTA counter epilogue), eager and CUDA-graph, with and without
// programmatic dependent launch (griddepcontrol.wait before the first global
// access) and with and without the cooperative attribute.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/pdl scripts/pdl_probe.cu && /tmp/pdl
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void __launch_bounds__(256, 1) k_copy(unsigned long long* ctrl, const uint4* src, uint4* dst,
                                                 long long nv, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  const long long T = (long long)gridDim.x * blockDim.x;
  for (long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x; j < nv; j += T) dst[j] = __ldcg(src + j);
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long prev = atomicAdd(ctrl + 1, 1ull);
    if (prev + 1 == gridDim.x) {
      ctrl[1] = 0;
      atomicAdd(ctrl, 1ull);
    }
  }
}

int main() {
  unsigned long long* ctrl;
  cudaMalloc(&ctrl, 64);
  cudaMemset(ctrl, 0, 64);
  const size_t maxb = 64 << 20;
  uint4 *src, *dst;
  cudaMalloc(&src, maxb);
  cudaMalloc(&dst, maxb);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_copy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t bytes : {size_t(16) << 10, size_t(1) << 20, size_t(8) << 20, size_t(32) << 20})
    for (int coop = 0; coop < 2; ++coop)
      for (int pdl = 0; pdl < 2; ++pdl) {
        auto launch = [&]() {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(148);
          cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = smem;
          cfg.stream = s;
          cudaLaunchAttribute at[2];
          int n = 0;
          if (coop) {
            at[n].id = cudaLaunchAttributeCooperative;
            at[n].val.cooperative = 1;
            ++n;
          }
          if (pdl) {
            at[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[n].val.programmaticStreamSerializationAllowed = 1;
            ++n;
          }
          cfg.attrs = at;
          cfg.numAttrs = n;
          return cudaLaunchKernelEx(&cfg, k_copy, ctrl, (const uint4*)src, dst, (long long)(bytes / 16), pdl);
        };
        const int reps = 200;
        // eager
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(a, s);
        for (int i = 0; i < reps; ++i) launch();
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms_e = 0;
        cudaEventElapsedTime(&ms_e, a, b);
        cudaError_t err = cudaGetLastError();
        // graph of 20
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int i = 0; i < 20; ++i) launch();
        cudaStreamEndCapture(s, &g);
        cudaGraphInstantiate(&ge, g, 0);
        for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, s);
        cudaEventRecord(a, s);
        for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms_g = 0;
        cudaEventElapsedTime(&ms_g, a, b);
        cudaError_t err2 = cudaGetLastError();
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
        printf("bytes=%9zu coop=%d pdl=%d: eager %.2f us/call  graph %.2f us/call  (%s / %s)\n", bytes, coop, pdl,
               ms_e * 1e3f / reps, ms_g * 1e3f / 200, cudaGetErrorString(err), cudaGetErrorString(err2));
      }
  return 0;
}
