#!/usr/bin/env python
"""Where the time goes in per-rank launches (cfg.launch_per_rank, BLINK_TRACE=1).

For m virtual ranks, each in its own launch, prints per rank the median over
its CTAs of every trace point relative to the earliest CTA start of ANY rank
(globaltimer, microseconds): launch skew, entry handshake, first load, stores
done, exit waits done.  Then times eager calls and CUDA-graph replays.
"""
import os
import statistics
import sys
import time

os.environ["BLINK_TRACE"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402

NAMES = ["start", "epoch", "entry", "1st-load", "1st-store", "stores", "exit", "end"]


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    sizes = [int(x) for x in sys.argv[2:]] or [1024, 1 << 20, 64 << 20]
    per_rank = int(os.environ.get("PER_RANK", "1"))
    comms = B.init_all([0] * m, cfg=B.config(launch_per_rank=per_rank, timeout_s=5.0))
    for nbytes in sizes:
        cnt = nbytes // 4
        xs = [torch.randn(cnt, device="cuda") for _ in range(m)]
        ys = [torch.empty_like(x) for x in xs]

        def call():
            for r, c in enumerate(comms):
                c.allreduce(xs[r], ys[r])
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        trs = [c.trace() for c in comms] if per_rank else [comms[0].trace()]
        t0 = min(t[0] for tr in trs for t in tr if t[0])
        print(f"m={m} bytes={nbytes}", flush=True)
        for r, tr in enumerate(trs):
            line = []
            for k, name in enumerate(NAMES):
                vals = [(t[k] - t0) / 1e3 for t in tr if t[k]]
                if vals:
                    line.append(f"{name}={statistics.median(vals):.1f}/{max(vals):.1f}")
            print(f"  rank {r} ctas={len(tr)}: " + " ".join(line), flush=True)
        last_start = max(min(t[0] for t in tr if t[0]) for tr in trs)
        end = max(max(t[7] for t in tr if t[7]) for tr in trs)
        print(f"  last rank start -> last CTA end: {(end - last_start) / 1e3:.1f} us", flush=True)
        n = 20
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t = time.perf_counter()
        e0.record()
        for _ in range(n):
            call()
        e1.record()
        torch.cuda.synchronize()
        print(f"  eager: {e0.elapsed_time(e1) / n * 1e3:.1f} us/call "
              f"(host {(time.perf_counter() - t) / n * 1e6:.1f} us/call)", flush=True)
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                call()
            g.replay()
            torch.cuda.synchronize()
            e0.record()
            for _ in range(n):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            print(f"  graph: {e0.elapsed_time(e1) / n * 1e3:.1f} us/call", flush=True)
        except Exception as ex:  # a replay that serialises the rank launches times out
            print(f"  graph: FAILED {ex}", flush=True)
            return


if __name__ == "__main__":
    main()
