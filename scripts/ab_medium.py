#!/usr/bin/env python
"""A/B helper: per-call device time (graph of 10 calls) of merged one-hop
AllReduce at medium sizes (1-48 MiB) for m = 8, 6, 4, 3, 2."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04940_b200 as B
from scripts.ab_env import per_call_us
for m in (8, 6, 4, 3, 2):
    comms = B.init_all([0] * m)
    out = []
    for mb in (1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48):
        n = (mb << 20) // 4
        xs = [torch.randn(n, device="cuda") for _ in range(m)]
        ys = [torch.empty_like(x) for x in xs]
        def fn():
            for r, c in enumerate(comms): c.allreduce(xs[r], ys[r])
        out.append(f"{mb}M:{per_call_us(fn, 20):.2f}")
    print(os.environ.get("BLINK_ONE_CHUNK", "1"), m, " ".join(out), flush=True)
    for c in comms: c.destroy()
