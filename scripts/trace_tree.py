#!/usr/bin/env python
"""BLINK_TRACE on a multi-hop config: per channel (rank, tree, role) the CTA
count and first-load / last-store times, to see where a multi-level plan waits."""
import os, sys, statistics
os.environ["BLINK_TRACE"] = "1"
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B
from oracle import graphs as OG

g = OG.dgx1v()
coll = sys.argv[1] if len(sys.argv) > 1 else "ar"
S = int(sys.argv[2]) if len(sys.argv) > 2 else 256 << 20
comms = B.init_all([0] * 8, graph=None if os.environ.get("SWITCH") else B.Graph.from_pairs(8, g[1]))
cnt = S // 4
xs = [torch.randn(cnt, device="cuda") for _ in range(8)]
ys = [torch.empty_like(x) for x in xs]
for _ in range(3):
    for r, c in enumerate(comms):
        if coll == "ar":
            c.allreduce(xs[r], ys[r])
        else:
            c.broadcast(xs[0] if r == 0 else None, ys[r], root=0)
torch.cuda.synchronize()
tr = comms[0].trace()
t0 = min(t[0] for t in tr)
plan = comms[0].plan(coll == "ar", 0, cnt)
print("trees:", [(t["root"], t["depth"], t["nchunks"]) for t in plan["trees"]], "ctas", len(tr))
ends = sorted(((t[5] - t0) / 1e3, i) for i, t in enumerate(tr) if t[5])
firsts = sorted(((t[3] - t0) / 1e3, i) for i, t in enumerate(tr) if t[3])
print("first-load: min/med/max", firsts[0][0], statistics.median(x for x, _ in firsts), firsts[-1][0])
print("stores-done: min/med/max", ends[0][0], statistics.median(x for x, _ in ends), ends[-1][0])
print("kernel end max", max((t[7] - t0) / 1e3 for t in tr))
if os.environ.get("PER_CTA"):
    for i, t in enumerate(tr):
        print(f"cta {i}: " + " ".join(f"{(x - t0) / 1e3:.1f}" if x else "-" for x in t[:8]))
