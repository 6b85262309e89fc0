import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04940_b200 as B
for m in (2, 8):
    comms = B.init_all([0] * m)
    xs = [torch.randn(256, device="cuda") for _ in range(m)]
    ys = [torch.empty_like(x) for x in xs]
    for _ in range(20):
        for r, c in enumerate(comms): c.allreduce(xs[r], ys[r])
    torch.cuda.synchronize()
    N = 2000
    t0 = time.perf_counter()
    for _ in range(N):
        for r, c in enumerate(comms): c.allreduce(xs[r], ys[r])
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"m={m}: host {1e6*(t1-t0)/N:.1f} us per collective ({1e6*(t1-t0)/N/m:.1f} per rank call), wall incl. drain {1e6*(t2-t0)/N:.1f} us")
    # raw ctypes floor: the same call with precomputed args
    lib = B._lib
    h = comms[0]._h
    import ctypes
    t0 = time.perf_counter()
    for _ in range(N):
        lib.blink_comm_info(h, None, None, None)
    t1 = time.perf_counter()
    print(f"  ctypes no-op call {1e6*(t1-t0)/N:.2f} us")
    for c in comms: c.destroy()

# breakdown (m = 8): Python marshalling vs the C call (C++ runtime + launch)
import ctypes
m = 8
comms = B.init_all([0] * m)
xs = [torch.randn(256, device="cuda") for _ in range(m)]
ys = [torch.empty_like(x) for x in xs]
for _ in range(20):
    for r, c in enumerate(comms): c.allreduce(xs[r], ys[r])
torch.cuda.synchronize()
N = 2000
sp, rp = [x.data_ptr() for x in xs], [y.data_ptr() for y in ys]
st = torch.cuda.current_stream().cuda_stream
lib = B._lib
t0 = time.perf_counter()
for _ in range(N):
    for r, c in enumerate(comms):
        lib.blink_allreduce(c._h, sp[r], rp[r], 256, 0, 0, st)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"m=8 direct C calls: {1e6*(t1-t0)/N:.1f} us per collective")
t0 = time.perf_counter()
for _ in range(N):
    for r, c in enumerate(comms):
        B._stream(None); B._dtype_of(xs[r], None); xs[r].numel(); xs[r].data_ptr(); ys[r].data_ptr()
t1 = time.perf_counter()
print(f"m=8 python marshalling only: {1e6*(t1-t0)/N:.1f} us per collective")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(200):
    for r, c in enumerate(comms): c.allreduce(xs[r], ys[r])
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(6)
