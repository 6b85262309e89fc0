import torch, time
n = 256 << 20
m = 8
h = [torch.empty(n // 4, dtype=torch.float32).pin_memory() for _ in range(m)]
hr = [torch.empty(n // 4, dtype=torch.float32).pin_memory() for _ in range(m)]
d = [torch.empty(n // 4, device="cuda") for _ in range(m)]
d2 = [torch.empty(n // 4, device="cuda") for _ in range(m)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps
def h2d():
    with torch.cuda.stream(s1):
        for r in range(m): d[r].copy_(h[r], non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        for r in range(m): hr[r].copy_(d2[r], non_blocking=True)
def both():
    h2d(); d2h()
a, b, c = t(h2d), t(d2h), t(both)
GB = m * n / 1e9
print(f"H2D {GB/a:.1f} GB/s, D2H {GB/b:.1f} GB/s, both concurrently: {2*GB/c:.1f} GB/s total ({c*1e3:.1f} ms for {GB:.2f} GB each way)")
