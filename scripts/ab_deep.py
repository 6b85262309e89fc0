#!/usr/bin/env python
"""Device time (graph replay) of the multi-hop configs at mid/large sizes."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.environ.get("AB_ROOT", os.getcwd()))
import paper_1910_04940_b200 as B
from oracle import graphs as OG

def run(comms, coll, S, root=0):
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
        for _ in range(10): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 100 * 1e3

g = OG.dgx1v()
tri, _ = OG.induced(OG.dgx1p(), [0, 1, 3])
cases = [("c1-bc", B.init_all([0]*3, graph=B.Graph.from_pairs(3, tri[1])), "bc"),
         ("c2-bc", B.init_all([0]*8, graph=B.Graph.from_pairs(8, g[1])), "bc"),
         ("c2-ar", None, "ar"),
         ("c3-bc", B.init_all([0]*8), "bc"),
         ("n4-44", B.init_all([0]*8, graph=B.Graph.multi_server(8, g[1], [[0,1,2,3],[4,5,6,7]])), "ar")]
cases[2] = ("c2-ar", cases[1][1], "ar")
line = []
only = os.environ.get("CASES")  # e.g. CASES=c2-bc,c2-ar
for name, comms, coll in cases:
    if only and name not in only.split(","):
        continue
    for S in (1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20):
        line.append(f"{name}/{S>>20}M:{run(comms, coll, S):.0f}")
print(os.environ.get("CFG_LABEL", os.environ.get("BLINK_MIN_CHUNK_DEEP", "default")), " ".join(line), flush=True)
