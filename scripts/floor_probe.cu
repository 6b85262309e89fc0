// Launch-floor probe: device time per call of near-empty kernels in the
// executor's launch shape (CUDA-graph replays, back to back), to separate the
// launch floor from the executor's own fixed cost.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/floor scripts/floor_probe.cu && /tmp/floor
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_empty() {}

// skeleton: thread 0 reads the epoch word, block barrier, last CTA advances it
__global__ void k_epoch(unsigned long long* ctrl) {
  __shared__ unsigned long long e;
  if (threadIdx.x == 0) e = *reinterpret_cast<volatile unsigned long long*>(ctrl) + 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long prev = atomicAdd(ctrl + 1, 1ull);
    if (prev + 1 == gridDim.x) {
      ctrl[1] = 0;
      atomicExch(ctrl, e);
    }
  }
}

// no load at entry: the last CTA increments the epoch
__global__ void k_counter(unsigned long long* ctrl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long prev = atomicAdd(ctrl + 1, 1ull);
    if (prev + 1 == gridDim.x) {
      ctrl[1] = 0;
      atomicAdd(ctrl, 1ull);
    }
  }
}

template <class F>
float graph_us(F launch, int reps) {
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < 20; ++i) launch(s);
  cudaStreamEndCapture(s, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int i = 0; i < 3; ++i) cudaGraphLaunch(ge, s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaStreamDestroy(s);
  return ms * 1e3f / (reps * 20);
}

int main() {
  unsigned long long* ctrl;
  cudaMalloc(&ctrl, 64);
  cudaMemset(ctrl, 0, 64);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k_empty, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_epoch, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k_counter, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (int coop = 0; coop < 2; ++coop)
    for (int grid : {8, 64, 148}) {
      for (int sm : {0, smem}) {
        auto mk = [&](auto fn, auto... args) {
          return [=](cudaStream_t s) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(256);
            cfg.dynamicSmemBytes = sm;
            cfg.stream = s;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = coop;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, fn, args...);
          };
        };
        float e0 = graph_us(mk(k_empty), 50);
        float e1 = graph_us(mk(k_epoch, ctrl), 50);
        float e2 = graph_us(mk(k_counter, ctrl), 50);
        printf("coop=%d grid=%3d smem=%6d: empty %.2f us  epoch-skeleton %.2f us  counter-skeleton %.2f us\n",
               coop, grid, sm, e0, e1, e2);
      }
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
