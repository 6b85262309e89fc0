#!/usr/bin/env python
"""DGX-1V Broadcast from root 0 (virtual ranks): device time per call,
graph replays of `per` calls, for per in (1, 10), at 1/16/64/256 MiB."""
import os, sys, torch
sys.path.insert(0, os.environ.get("AB_ROOT", os.getcwd()))
import paper_1910_04940_b200 as B
from oracle import graphs as OG


def run(comms, coll, S, per, root=0):
    m = len(comms); cnt = S // 4
    xs = [torch.randn(cnt, device="cuda") for _ in range(m)]
    ys = [torch.empty_like(x) for x in xs]
    def fn():
        for r, c in enumerate(comms):
            if coll == "ar": c.allreduce(xs[r], ys[r])
            else: c.broadcast(xs[root] if r == root else None, ys[r], root=root)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(per): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (10 * per) * 1e3


g = OG.dgx1v()
# EXTRA=k: k other 8-rank switch comms stay alive on the device first
extra = [B.init_all([0] * 8) for _ in range(int(os.environ.get("EXTRA", "0")))]
if os.environ.get("EXTRA_FIRST_ONLY"):
    for cs in extra:
        for c in cs:
            c.destroy()
    extra = []
comms = B.init_all([0] * 8, graph=B.Graph.from_pairs(8, g[1]))
coll = sys.argv[1] if len(sys.argv) > 1 else "bc"
line = []
for S in (1 << 20, 16 << 20, 64 << 20, 256 << 20):
    for per in (1, 10):
        line.append(f"{S >> 20}M/x{per}:{run(comms, coll, S, per):.0f}")
print(os.environ.get("CFG_LABEL", ""), coll, " ".join(line), flush=True)
