// NEXT-1 host side: NVLS multicast objects for the one-hop trees in the
// switch (kernel and protocol: nvls.cu).
//
// Every rank binds `bytes` of its own physical memory to one multicast object
// and maps it twice: unicast (its own copy) and multicast (the switch
// address: multimem.ld_reduce reads every rank's copy, multimem.st writes
// every rank's copy).  All devices must join the object before any memory is
// bound to it.
//   single process (init_all, one rank per device): create, add every device,
//     then bind + map per device;
//   one process per GPU: rank 0 creates the object at blink_init and exports
//     it in its blob -- a FABRIC handle where the device supports them (IMEX
//     / fabric manager), else a POSIX fd that the peers duplicate from rank
//     0's process with pidfd_getfd (one node, same user); at blink_connect
//     every rank imports it and adds its device, the ranks meet at a barrier
//     in each other's flag words, bind + map, and meet again; NVLS turns on
//     only if every rank succeeded.
// Driver symbols come from cudaGetDriverEntryPoint (the library never links
// libcuda).
#include <cuda.h>
#include <cuda_runtime.h>

#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "blink_internal.h"

namespace blink {
namespace {

struct Drv {
  bool ok = false;
  std::string err;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetAttribute)(int*, CUdevice_attribute, CUdevice) = nullptr;
  CUresult (*MulticastCreate)(CUmemGenericAllocationHandle*, const CUmulticastObjectProp*) = nullptr;
  CUresult (*MulticastAddDevice)(CUmemGenericAllocationHandle, CUdevice) = nullptr;
  CUresult (*MulticastBindMem)(CUmemGenericAllocationHandle, size_t, CUmemGenericAllocationHandle, size_t, size_t,
                               unsigned long long) = nullptr;
  CUresult (*MulticastUnbind)(CUmemGenericAllocationHandle, CUdevice, size_t, size_t) = nullptr;
  CUresult (*MulticastGetGranularity)(size_t*, const CUmulticastObjectProp*,
                                      CUmulticastGranularity_flags) = nullptr;
  CUresult (*MemCreate)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                        unsigned long long) = nullptr;
  CUresult (*MemRelease)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*MemAddressReserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*MemAddressFree)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemMap)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long) = nullptr;
  CUresult (*MemUnmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*MemSetAccess)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t) = nullptr;
  CUresult (*MemExportToShareableHandle)(void*, CUmemGenericAllocationHandle, CUmemAllocationHandleType,
                                         unsigned long long) = nullptr;
  CUresult (*MemImportFromShareableHandle)(CUmemGenericAllocationHandle*, void*, CUmemAllocationHandleType) = nullptr;
  CUresult (*MemRetainAllocationHandle)(CUmemGenericAllocationHandle*, void*) = nullptr;
  CUresult (*MemGetAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
};

template <class F>
bool load(const char* name, F* out, std::string* err) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qr;
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &qr) != cudaSuccess || !fn) {
    cudaGetLastError();
    *err = std::string("driver entry point ") + name + " not found";
    return false;
  }
  *out = reinterpret_cast<F>(fn);
  return true;
}

const Drv& drv() {
  static Drv d = [] {
    Drv x;
    std::string& e = x.err;
    x.ok = load("cuDeviceGet", &x.DeviceGet, &e) && load("cuDeviceGetAttribute", &x.DeviceGetAttribute, &e) &&
           load("cuMulticastCreate", &x.MulticastCreate, &e) &&
           load("cuMulticastAddDevice", &x.MulticastAddDevice, &e) &&
           load("cuMulticastBindMem", &x.MulticastBindMem, &e) &&
           load("cuMulticastUnbind", &x.MulticastUnbind, &e) &&
           load("cuMulticastGetGranularity", &x.MulticastGetGranularity, &e) &&
           load("cuMemCreate", &x.MemCreate, &e) && load("cuMemRelease", &x.MemRelease, &e) &&
           load("cuMemAddressReserve", &x.MemAddressReserve, &e) &&
           load("cuMemAddressFree", &x.MemAddressFree, &e) && load("cuMemMap", &x.MemMap, &e) &&
           load("cuMemUnmap", &x.MemUnmap, &e) && load("cuMemSetAccess", &x.MemSetAccess, &e) &&
           load("cuMemExportToShareableHandle", &x.MemExportToShareableHandle, &e) &&
           load("cuMemImportFromShareableHandle", &x.MemImportFromShareableHandle, &e) &&
           load("cuMemRetainAllocationHandle", &x.MemRetainAllocationHandle, &e) &&
           load("cuMemGetAddressRange", &x.MemGetAddressRange, &e);
    return x;
  }();
  return d;
}

#define DRV_TRY(call, what)                                       \
  do {                                                            \
    CUresult r_ = (call);                                         \
    if (r_ != CUDA_SUCCESS) {                                     \
      *err = std::string(what) + " failed (CUresult " + std::to_string(int(r_)) + ")"; \
      return false;                                               \
    }                                                             \
  } while (0)

CUmulticastObjectProp mc_prop(int ndev, size_t bytes, CUmemAllocationHandleType ht) {
  CUmulticastObjectProp p;
  memset(&p, 0, sizeof p);
  p.numDevices = unsigned(ndev);
  p.size = bytes;
  p.handleTypes = ht;
  return p;
}

}  // namespace

CUmemAllocationHandleType handle_type(int share) {
  return share == kNvlsFabric ? CU_MEM_HANDLE_TYPE_FABRIC
                              : (share == kNvlsPosixFd ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
                                                       : CU_MEM_HANDLE_TYPE_NONE);
}

bool nvls_fabric_supported(int dev) {
  const Drv& d = drv();
  CUdevice cd;
  int fab = 0;
  if (!d.ok || d.DeviceGet(&cd, dev) != CUDA_SUCCESS) return false;
  d.DeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, cd);
  return fab != 0;
}

bool nvls_supported(int dev, int share, std::string* err) {
  const bool fabric = share == kNvlsFabric;
  const Drv& d = drv();
  if (!d.ok) {
    *err = d.err;
    return false;
  }
  CUdevice cd;
  DRV_TRY(d.DeviceGet(&cd, dev), "cuDeviceGet");
  int mc = 0, fab = 0;
  DRV_TRY(d.DeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cd), "cuDeviceGetAttribute");
  if (!mc) {
    *err = "device " + std::to_string(dev) + " does not support multicast (NVLS)";
    return false;
  }
  if (fabric) {
    d.DeviceGetAttribute(&fab, CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED, cd);
    if (!fab) {
      *err = "device " + std::to_string(dev) + " cannot export FABRIC handles (multi-process NVLS)";
      return false;
    }
  }
  return true;
}

// size rounded up to the multicast granularity
size_t nvls_round(int ndev, size_t bytes) {
  const Drv& d = drv();
  size_t g = size_t(2) << 20;
  if (d.ok) {
    CUmulticastObjectProp p = mc_prop(ndev, bytes, CU_MEM_HANDLE_TYPE_NONE);
    size_t r = 0;
    if (d.MulticastGetGranularity(&r, &p, CU_MULTICAST_GRANULARITY_RECOMMENDED) == CUDA_SUCCESS && r) g = r;
  }
  return (bytes + g - 1) / g * g;
}

bool nvls_create(int ndev, size_t bytes, int share, NvlsMem* m, std::string* err) {
  const Drv& d = drv();
  CUmulticastObjectProp p = mc_prop(ndev, bytes, handle_type(share));
  CUmemGenericAllocationHandle h;
  DRV_TRY(d.MulticastCreate(&h, &p), "cuMulticastCreate");
  m->mc = h;
  m->size = bytes;
  m->owner = true;
  m->share = share;
  return true;
}

bool nvls_export(NvlsMem* m, void* handle, std::string* err) {
  const Drv& d = drv();
  if (m->share == kNvlsPosixFd) {
    if (m->export_fd < 0) {
      int fd = -1;
      DRV_TRY(d.MemExportToShareableHandle(&fd, m->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
              "cuMemExportToShareableHandle(POSIX_FD)");
      m->export_fd = fd;  // stays open until release: peers duplicate it with pidfd_getfd
    }
    memcpy(handle, &m->export_fd, sizeof m->export_fd);
    return true;
  }
  DRV_TRY(d.MemExportToShareableHandle(handle, m->mc, CU_MEM_HANDLE_TYPE_FABRIC, 0),
          "cuMemExportToShareableHandle(FABRIC)");
  return true;
}

bool nvls_import(const void* handle, int share, size_t bytes, NvlsMem* m, std::string* err) {
  const Drv& d = drv();
  CUmemGenericAllocationHandle h;
  if (share == kNvlsPosixFd) {
    int fd = -1;
    memcpy(&fd, handle, sizeof fd);
    DRV_TRY(d.MemImportFromShareableHandle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(fd)),
                                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
            "cuMemImportFromShareableHandle(POSIX_FD)");
  } else {
    DRV_TRY(d.MemImportFromShareableHandle(&h, const_cast<void*>(handle), CU_MEM_HANDLE_TYPE_FABRIC),
            "cuMemImportFromShareableHandle(FABRIC)");
  }
  m->mc = h;
  m->size = bytes;
  m->owner = true;  // this process's reference
  m->share = share;
  return true;
}

bool nvls_add_device(NvlsMem* m, int dev, std::string* err) {
  const Drv& d = drv();
  CUdevice cd;
  DRV_TRY(d.DeviceGet(&cd, dev), "cuDeviceGet");
  DRV_TRY(d.MulticastAddDevice(m->mc, cd), "cuMulticastAddDevice");
  m->dev = dev;
  return true;
}

// after every device joined: bind this device's memory and map uc + mc
bool nvls_bind_map(NvlsMem* m, int dev, std::string* err) {
  const Drv& d = drv();
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof ap);
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = dev;
  ap.requestedHandleTypes = handle_type(m->share);
  DRV_TRY(d.MemCreate(&m->mem, m->size, &ap, 0), "cuMemCreate");
  DRV_TRY(d.MulticastBindMem(m->mc, 0, m->mem, 0, m->size, 0), "cuMulticastBindMem");
  m->bound = true;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  const size_t align = size_t(2) << 20;
  DRV_TRY(d.MemAddressReserve(&m->uc_va, m->size, align, 0, 0), "cuMemAddressReserve(uc)");
  DRV_TRY(d.MemMap(m->uc_va, m->size, 0, m->mem, 0), "cuMemMap(uc)");
  DRV_TRY(d.MemSetAccess(m->uc_va, m->size, &acc, 1), "cuMemSetAccess(uc)");
  DRV_TRY(d.MemAddressReserve(&m->mc_va, m->size, align, 0, 0), "cuMemAddressReserve(mc)");
  DRV_TRY(d.MemMap(m->mc_va, m->size, 0, m->mc, 0), "cuMemMap(mc)");
  DRV_TRY(d.MemSetAccess(m->mc_va, m->size, &acc, 1), "cuMemSetAccess(mc)");
  return true;
}

void nvls_release(NvlsMem* m) {
  const Drv& d = drv();
  if (!d.ok) return;
  if (m->mc_va) {
    d.MemUnmap(m->mc_va, m->size);
    d.MemAddressFree(m->mc_va, m->size);
  }
  if (m->uc_va) {
    d.MemUnmap(m->uc_va, m->size);
    d.MemAddressFree(m->uc_va, m->size);
  }
  if (m->bound) {
    CUdevice cd;
    if (d.DeviceGet(&cd, m->dev) == CUDA_SUCCESS) d.MulticastUnbind(m->mc, cd, 0, m->size);
  }
  if (m->mem) d.MemRelease(m->mem);
  if (m->mc && m->owner) d.MemRelease(m->mc);  // one reference per process
  if (m->export_fd >= 0) close(m->export_fd);
  *m = NvlsMem();
}

bool nvls_setup_single(const std::vector<int>& devs, size_t bytes, std::vector<NvlsMem>* out,
                       std::string* err) {
  const int n = int(devs.size());
  for (int dv : devs)
    if (!nvls_supported(dv, kNvlsLocal, err)) return false;
  int cur = 0;
  cudaGetDevice(&cur);
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{cur};
  const size_t size = nvls_round(n, bytes);
  NvlsMem base;
  if (!nvls_create(n, size, kNvlsLocal, &base, err)) return false;
  out->assign(n, NvlsMem());
  for (int i = 0; i < n; ++i) {
    if (!nvls_add_device(&base, devs[i], err)) {
      nvls_release(&base);
      return false;
    }
  }
  for (int i = 0; i < n; ++i) {
    NvlsMem& m = (*out)[i];
    m.mc = base.mc;      // one object, mapped on every device
    m.size = size;
    m.dev = devs[i];
    m.owner = i == 0;
    cudaSetDevice(devs[i]);
    if (!nvls_bind_map(&m, devs[i], err)) return false;
  }
  return true;
}

// ------------------------------------------------------------ VMM registration
// PyTorch's expandable segments map fixed-size physical chunks (cuMemCreate,
// POSIX-fd exportable) into one reserved range; a tensor can straddle chunks.
// The legacy cudaIpcGetMemHandle rejects such memory, so registration exports
// every chunk the buffer touches and the peers map them back to back.
bool vmm_chunks(const void* buf, size_t bytes, std::vector<VmmChunk>* out, std::string* err) {
  const Drv& d = drv();
  if (!d.ok) {
    *err = d.err;
    return false;
  }
  out->clear();
  const CUdeviceptr b = reinterpret_cast<CUdeviceptr>(buf);
  CUdeviceptr a = b;
  while (a < b + bytes) {
    CUdeviceptr cb = 0;
    size_t cs = 0;
    DRV_TRY(d.MemGetAddressRange(&cb, &cs, a), "cuMemGetAddressRange");
    CUmemGenericAllocationHandle h;
    DRV_TRY(d.MemRetainAllocationHandle(&h, reinterpret_cast<void*>(cb)), "cuMemRetainAllocationHandle");
    int fd = -1;
    CUresult r = d.MemExportToShareableHandle(&fd, h, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    d.MemRelease(h);
    if (r != CUDA_SUCCESS) {
      *err = "cuMemExportToShareableHandle(POSIX fd) failed (CUresult " + std::to_string(int(r)) +
             "): the allocation is not exportable";
      return false;
    }
    VmmChunk c;
    c.off = int64_t(cb) - int64_t(b);
    c.size = cs;
    c.fd = fd;
    out->push_back(c);
    a = cb + cs;
  }
  return true;
}

bool vmm_map_peer(const std::vector<VmmChunk>& chunks, const std::vector<int>& local_fds, int dev,
                  VmmMapping* out, std::string* err) {
  const Drv& d = drv();
  if (!d.ok) {
    *err = d.err;
    return false;
  }
  if (chunks.empty()) {
    *err = "no chunks";
    return false;
  }
  const int64_t first = chunks.front().off;
  const int64_t span = chunks.back().off + int64_t(chunks.back().size) - first;
  CUdeviceptr va = 0;
  DRV_TRY(d.MemAddressReserve(&va, size_t(span), size_t(2) << 20, 0, 0), "cuMemAddressReserve");
  out->va = va;
  out->span = size_t(span);
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof acc);
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  for (size_t i = 0; i < chunks.size(); ++i) {
    CUmemGenericAllocationHandle h;
    DRV_TRY(d.MemImportFromShareableHandle(&h, reinterpret_cast<void*>(static_cast<intptr_t>(local_fds[i])),
                                           CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
            "cuMemImportFromShareableHandle(POSIX fd)");
    const CUdeviceptr at = va + CUdeviceptr(chunks[i].off - first);
    CUresult r = d.MemMap(at, chunks[i].size, 0, h, 0);
    d.MemRelease(h);  // the mapping keeps the memory alive
    if (r != CUDA_SUCCESS) {
      *err = "cuMemMap of a peer chunk failed (CUresult " + std::to_string(int(r)) + ")";
      return false;
    }
    out->mapped.push_back({at, chunks[i].size});
    DRV_TRY(d.MemSetAccess(at, chunks[i].size, &acc, 1), "cuMemSetAccess");
  }
  out->base = reinterpret_cast<char*>(va) - first;  // the peer's buf
  return true;
}

void vmm_unmap(VmmMapping* m) {
  const Drv& d = drv();
  if (!d.ok) return;
  for (auto& x : m->mapped) d.MemUnmap(x.first, x.second);
  if (m->va) d.MemAddressFree(m->va, m->span);
  *m = VmmMapping();
}

}  // namespace blink
