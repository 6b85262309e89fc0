#!/usr/bin/env python
"""A/B helper: per-call device time of multi-level AllReduce plans (DGX-1V, two
fragments, 3+5 emulated servers) at 1-256 MiB (graph of 4 calls)."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1910_04940_b200 as B
from oracle import graphs as OG
from scripts.ab_env import per_call_us
g = OG.dgx1v()
cfgs = [("c2ar", 8, B.Graph.from_pairs(8, g[1]))]
for nodes in ([0, 1, 3, 4, 5, 7], [1, 4, 5, 6]):
    sub, _ = OG.induced(g, nodes)
    cfgs.append((f"frag{len(nodes)}", len(nodes), B.Graph.from_pairs(len(nodes), sub[1])))
cfgs.append(("ms3+5", 8, B.Graph.multi_server(8, g[1], [[0, 1, 2], [3, 4, 5, 6, 7]])))
for name, m, G in cfgs:
    comms = B.init_all([0] * m, graph=G)
    out = []
    for nbytes in (1 << 20, 16 << 20, 64 << 20, 256 << 20):
        xs = [torch.randn(nbytes // 4, device="cuda") for _ in range(m)]
        ys = [torch.empty_like(x) for x in xs]
        def fn():
            for r, c in enumerate(comms): c.allreduce(xs[r], ys[r])
        us = per_call_us(fn, 5 if nbytes <= (16 << 20) else 2, per_graph=4)
        out.append(f"{nbytes >> 20}M:{us:.1f}")
    print(os.environ.get("CFG_LABEL", ""), name, " ".join(out), flush=True)
    for c in comms: c.destroy()
