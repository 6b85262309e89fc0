// NVLS (NVSwitch multicast) probe for a single B200 behind an NVSwitch fabric.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/nvls_probe scripts/nvls_probe.cu -lcuda
//   /tmp/nvls_probe [MiB]
//
// 1. Reports CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and the multicast granularity.
// 2. Creates a multicast object with one device, binds device memory to it and
//    maps both the unicast and the multicast address.
// 3. Checks multimem.st (writes through the switch land in the bound memory) and
//    multimem.ld_reduce (a one-member reduction returns the value itself).
// 4. Times plain st.global, multimem.st and multimem.ld_reduce over the buffer:
//    multicast traffic leaves the GPU over NVLink to the switch and comes back,
//    so this is the one NVLink-port measurement a single-GPU box can make.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s_; cuGetErrorString(r_, &s_); \
  printf("FAIL %s: %s (%d)\n", #x, s_, int(r_)); return 1; } } while (0)
#define CR(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("FAIL %s: %s\n", #x, cudaGetErrorString(r_)); return 1; } } while (0)

__global__ void st_plain(float4* p, size_t n, float v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    p[i] = make_float4(v, v + 1, v + 2, v + 3);
}
__global__ void st_mc(float4* mc, size_t n, float v) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    asm volatile("multimem.st.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc + i), "f"(v), "f"(v + 1), "f"(v + 2),
                 "f"(v + 3) : "memory");
}
__global__ void ldred_mc(const float4* mc, float4* out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(mc + i) : "memory");
    out[i] = make_float4(a, b, c, d);
  }
}
__global__ void ld_plain(const float4* src, float4* out, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    out[i] = __ldcg(src + i);
}

int main(int argc, char** argv) {
  size_t mib = argc > 1 ? strtoull(argv[1], 0, 10) : 1024;
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CR(cudaSetDevice(0));
  CR(cudaFree(0));
  int mc_ok = 0, fab = 0;
  CK(cuDeviceGetAttribute(&mc_ok, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
  cuDeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, dev);
  printf("multicast_supported=%d fabric_handle_supported=%d\n", mc_ok, fab);
  if (!mc_ok) return 0;

  CUmulticastObjectProp mp;
  memset(&mp, 0, sizeof mp);
  mp.numDevices = 1;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  mp.size = mib << 20;
  size_t gmin = 0, grec = 0;
  CK(cuMulticastGetGranularity(&gmin, &mp, CU_MULTICAST_GRANULARITY_MINIMUM));
  CK(cuMulticastGetGranularity(&grec, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t size = ((mib << 20) + grec - 1) / grec * grec;
  mp.size = size;
  printf("granularity min=%zu recommended=%zu size=%zu\n", gmin, grec, size);
  CUmemGenericAllocationHandle mc;
  // handle types: POSIX fd (single node), FABRIC (IMEX), none
  const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                            CU_MEM_HANDLE_TYPE_FABRIC, CU_MEM_HANDLE_TYPE_NONE};
  CUmemAllocationHandleType ht = CU_MEM_HANDLE_TYPE_NONE;
  CUresult cr = CUDA_ERROR_UNKNOWN;
  const size_t sizes[3] = {size, gmin, grec};
  for (int j = 0; j < 3 && cr != CUDA_SUCCESS; ++j)
    for (int i = 0; i < 3; ++i) {
      mp.handleTypes = hts[i];
      mp.size = sizes[j];
      cr = cuMulticastCreate(&mc, &mp);
      const char* es = "";
      cuGetErrorString(cr, &es);
      printf("cuMulticastCreate(numDevices=1, size=%zu, handleTypes=%d) -> %d %s\n", sizes[j], int(hts[i]),
             int(cr), es);
      if (cr == CUDA_SUCCESS) {
        ht = hts[i];
        size = sizes[j];
        break;
      }
    }
  if (cr != CUDA_SUCCESS) return 1;
  CK(cuMulticastAddDevice(mc, dev));

  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = ht;
  CUmemGenericAllocationHandle mem;
  CK(cuMemCreate(&mem, size, &ap, 0));
  CK(cuMulticastBindMem(mc, 0, mem, 0, size, 0));

  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = 0;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUdeviceptr uc_va, mc_va;
  CK(cuMemAddressReserve(&uc_va, size, grec, 0, 0));
  CK(cuMemMap(uc_va, size, 0, mem, 0));
  CK(cuMemSetAccess(uc_va, size, &acc, 1));
  CK(cuMemAddressReserve(&mc_va, size, grec, 0, 0));
  CK(cuMemMap(mc_va, size, 0, mc, 0));
  CK(cuMemSetAccess(mc_va, size, &acc, 1));
  printf("mapped uc=%p mc=%p\n", (void*)uc_va, (void*)mc_va);

  const size_t n = size / 16;
  float4* uc = reinterpret_cast<float4*>(uc_va);
  float4* mcp = reinterpret_cast<float4*>(mc_va);
  float4* out;
  CR(cudaMalloc(&out, size));
  const int grid = 148 * 4, blk = 512;

  // correctness
  st_mc<<<grid, blk>>>(mcp, n, 3.0f);
  CR(cudaDeviceSynchronize());
  float h[8];
  CR(cudaMemcpy(h, uc + (n - 2), 32, cudaMemcpyDeviceToHost));
  printf("multimem.st -> unicast tail: %g %g %g %g (want 3 4 5 6)\n", h[4], h[5], h[6], h[7]);
  st_plain<<<grid, blk>>>(uc, n, 7.0f);
  ldred_mc<<<grid, blk>>>(mcp, out, n);
  CR(cudaDeviceSynchronize());
  CR(cudaMemcpy(h, out + 5, 16, cudaMemcpyDeviceToHost));
  printf("multimem.ld_reduce (1 member): %g %g %g %g (want 7 8 9 10)\n", h[0], h[1], h[2], h[3]);
  int bad = (h[0] != 7.f || h[3] != 10.f);

  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char* name, auto launch, double bytes) {
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    const int reps = 10;
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-28s %8.3f ms  %8.1f GB/s\n", name, ms, bytes / (ms * 1e-3) / 1e9);
  };
  timeit("st.global (HBM write)", [&] { st_plain<<<grid, blk>>>(uc, n, 1.f); }, double(size));
  timeit("multimem.st (via switch)", [&] { st_mc<<<grid, blk>>>(mcp, n, 1.f); }, double(size));
  timeit("ld.global.cg + st", [&] { ld_plain<<<grid, blk>>>(uc, out, n); }, double(size));
  timeit("multimem.ld_reduce + st", [&] { ldred_mc<<<grid, blk>>>(mcp, out, n); }, double(size));
  CR(cudaGetLastError());
  printf(bad ? "NVLS probe: WRONG VALUES\n" : "NVLS probe: ok\n");
  return bad;
}
