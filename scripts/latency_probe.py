#!/usr/bin/env python
"""Small-message latency: host enqueue cost vs device time per call.

For m virtual ranks and tiny buffers, prints
  host_us   : wall time to enqueue one call (m binding calls incl. launch)
  gpu_us    : CUDA-event time per call when the host runs far ahead
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402


def main():
    s = torch.cuda.current_stream()
    for m in (2, 8):
        comms = B.init_all([0] * m)
        for nbytes in (1024, 1 << 20, 16 << 20):
            cnt = nbytes // 4
            xs = [torch.randn(cnt, device="cuda") for _ in range(m)]
            ys = [torch.empty_like(x) for x in xs]
            ptrs = [(x.data_ptr(), y.data_ptr()) for x, y in zip(xs, ys)]
            sp = s.cuda_stream

            def call():
                for r, c in enumerate(comms):
                    c.allreduce(ptrs[r][0], ptrs[r][1], count=cnt, dtype="f32", stream=sp)
            for _ in range(5):
                call()
            torch.cuda.synchronize()
            n = 200
            t0 = time.perf_counter()
            for _ in range(n):
                call()
            t1 = time.perf_counter()
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            host_us = (t1 - t0) / n * 1e6
            # device-only: block the stream first so the host runs ahead
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda._sleep(int(2e8))
            e0.record()
            for _ in range(n):
                call()
            e1.record()
            torch.cuda.synchronize()
            gpu_us = e0.elapsed_time(e1) / n * 1e3
            print(f"m={m} bytes={nbytes}: host_us/call={host_us:.1f} wall_us/call={(t2 - t0) / n * 1e6:.1f} "
                  f"gpu_us/call={gpu_us:.1f}", flush=True)
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
