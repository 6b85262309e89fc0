#!/usr/bin/env python
"""A/B of environment knobs: device time per call (CUDA-graph replays) of
config-3 AllReduce and Broadcast (m = 8 virtual ranks, fp32) over sizes.

    CFG_LABEL=x BLINK_MIN_CHUNK=4096 python scripts/ab_env.py [ar|bc|both]
"""
import os
import sys

import torch

# AB_ROOT: import the package from another checkout (A/B of builds)
sys.path.insert(0, os.environ.get("AB_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1910_04940_b200 as B  # noqa: E402

SIZES = (256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20)


def per_call_us(fn, reps, per_graph=10):
    """Device time per call: `per_graph` back-to-back calls captured in one
    CUDA graph (a graph launch has its own fixed cost), replayed `reps` times."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(per_graph):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (reps * per_graph) * 1e3


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "both"
    m = 8
    comms = B.init_all([0] * m)
    for coll in (("ar", "bc") if which == "both" else (which,)):
        out = []
        for nbytes in SIZES:
            cnt = nbytes // 4
            xs = [torch.randn(cnt, device="cuda") for _ in range(m)]
            ys = [torch.empty_like(x) for x in xs]

            def fn():
                for r, c in enumerate(comms):
                    if coll == "ar":
                        c.allreduce(xs[r], ys[r])
                    else:
                        c.broadcast(xs[0] if r == 0 else None, ys[r], root=0)
            us = per_call_us(fn, 20 if nbytes <= (16 << 20) else 3)
            out.append(f"{nbytes >> 10}K:{us:.1f}")
            del xs, ys
        print(f"{os.environ.get('CFG_LABEL', '')} {coll} " + " ".join(out), flush=True)


if __name__ == "__main__":
    main()
