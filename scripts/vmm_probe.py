import ctypes, os
os.environ["PYTORCH_CUDA_ALLOC_CONF"] = "expandable_segments:True"
import torch
cuda = ctypes.CDLL("libcuda.so.1")
x = torch.empty(50 << 20, dtype=torch.uint8, device="cuda")   # 50 MiB
y = torch.empty(30 << 20, dtype=torch.uint8, device="cuda")
for name, t in (("x", x), ("y", y), ("y+25M", y[25 << 20:])):
    p = ctypes.c_uint64(t.data_ptr())
    base = ctypes.c_uint64(); size = ctypes.c_size_t()
    r = cuda.cuMemGetAddressRange_v2(ctypes.byref(base), ctypes.byref(size), p)
    h = ctypes.c_uint64()
    r2 = cuda.cuMemRetainAllocationHandle(ctypes.byref(h), ctypes.c_void_p(t.data_ptr()))
    fd = ctypes.c_int(-1)
    r3 = cuda.cuMemExportToShareableHandle(ctypes.byref(fd), h, 1, 0) if r2 == 0 else -1
    print(name, hex(t.data_ptr()), "range r", r, hex(base.value), size.value >> 20, "MiB", "retain", r2, "export", r3, fd.value)
# legacy IPC handle on it
class H(ctypes.Structure):
    _fields_ = [("r", ctypes.c_char * 64)]
rt = torch.cuda.cudart()
try:
    h = torch.cuda._get_device_properties  # noqa
except Exception:
    pass
lib = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
if lib:
    hh = H()
    print("cudaIpcGetMemHandle", lib.cudaIpcGetMemHandle(ctypes.byref(hh), ctypes.c_void_p(x.data_ptr())))
