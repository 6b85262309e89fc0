#!/usr/bin/env python
"""Per-hop latency of the tree executor: Broadcast of ONE chunk down a path
0 -> 1 -> ... -> m-1 (virtual ranks, LL and the shallow tree off), device time
per call of 10 back-to-back calls in a CUDA graph, for m = 2..8.  The slope
over the path length is the cost of one hop (flag wait -> TMA load -> bulk
store -> completion -> flag), the intercept the launch / entry / exit cost.

    CFG_LABEL=x [BLINK_...] python scripts/hop_probe.py [chunk bytes, default 16384]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.environ.get("AB_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402  (topology presets only)

nbytes = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
xs, ys = [], []
for m in range(2, 9):
    g = OG.from_pairs(m, [(i, i + 1) for i in range(m - 1)])
    comms = B.init_all([0] * m, graph=B.Graph.from_pairs(m, g[1]),
                       cfg=B.config(chunk_bytes=nbytes, ll_max_bytes=0, shallow_max_bytes=0, timeout_s=10.0))
    cnt = nbytes // 4
    src = torch.randn(cnt, device="cuda")
    out = [torch.empty_like(src) for _ in range(m)]

    def fn():
        for r, c in enumerate(comms):
            c.broadcast(src if r == 0 else None, out[r], root=0)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g_ = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_):
        for _ in range(10):
            fn()
    g_.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        g_.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 200 * 1e3
    assert torch.equal(out[-1], src)
    assert comms[0].stats()["last_chunks"] == 1, comms[0].stats()
    xs.append(m - 1)
    ys.append(us)
    for c in comms:
        c.destroy()
slope, icpt = np.polyfit(xs, ys, 1)
print(f"{os.environ.get('CFG_LABEL', ''):10s} chunk {nbytes}: " + " ".join(f"h{h}:{u:.2f}" for h, u in zip(xs, ys)) +
      f"  -> {slope:.2f} us/hop + {icpt:.2f} us", flush=True)
