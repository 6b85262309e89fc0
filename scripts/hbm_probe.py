#!/usr/bin/env python
"""Calibrate attainable HBM bandwidth on this box for read+write streams.

Prints GB/s (read+write bytes / time, like MEASURED_PEAKS.json hbm_gbs) for:
  torch copy_            2 GiB -> 2 GiB
  torch sum of 8 tensors (8 x 256 MiB read, 256 MiB written)
  blink m=2 Broadcast star, m=8 AllReduce, m=2 AllReduce (virtual ranks)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402


def timeit(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    n = 1 << 29  # 2 GiB fp32
    a = torch.randn(n, device="cuda")
    b = torch.empty_like(a)
    t = timeit(lambda: b.copy_(a))
    print(f"torch copy_ 2GiB: {2 * a.numel() * 4 / t / 1e9:.0f} GB/s")
    xs = [torch.randn(1 << 26, device="cuda") for _ in range(8)]
    out = torch.empty_like(xs[0])

    def s8():
        torch.sum(torch.stack(xs), 0, out=out)
    t = timeit(s8, 5)
    print(f"torch stack+sum 8x256MiB (incl. stack copy): {(9 * xs[0].numel() * 4) / t / 1e9:.0f} GB/s (alg 9S)")
    for m in (2, 4, 8):
        comms = B.init_all([0] * m)
        cnt = (1 << 31) // 4 // m  # total send bytes 2 GiB
        sends = [torch.randn(cnt, device="cuda") for _ in range(m)]
        recvs = [torch.empty_like(s) for s in sends]

        def ar():
            for r, c in enumerate(comms):
                c.allreduce(sends[r], recvs[r])
        t = timeit(ar)
        print(f"blink allreduce m={m} S={cnt * 4 >> 20}MiB: HBM {2 * m * cnt * 4 / t / 1e9:.0f} GB/s, algBW {cnt * 4 / t / 1e9:.0f}")

        def bc():
            for r, c in enumerate(comms):
                c.broadcast(sends[0] if r == 0 else None, recvs[r], root=0)
        t = timeit(bc)
        # root reads S (+ inner nodes re-read), writes m*S (own recv + m-1 peers)
        print(f"blink broadcast m={m}: algBW {cnt * 4 / t / 1e9:.0f} GB/s, HBM>= {(m + 1) * cnt * 4 / t / 1e9:.0f}")
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
