#!/usr/bin/env python
"""BLINK_TRACE of one chunk down the path 0 -> ... -> 7 (scripts/hop_probe.py's
case): per CTA (one per hop) the trace stamps relative to the first CTA's
start -- 0 start, 1 epoch, 2 setup, 3 first TMA load, 4 first bulk store,
5 last stores complete, 6 end of work, 7 after the epoch update."""
import os
import sys

os.environ["BLINK_TRACE"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402

nbytes = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m = 8
g = OG.from_pairs(m, [(i, i + 1) for i in range(m - 1)])
comms = B.init_all([0] * m, graph=B.Graph.from_pairs(m, g[1]),
                   cfg=B.config(chunk_bytes=nbytes, ll_max_bytes=0, shallow_max_bytes=0, timeout_s=10.0))
src = torch.randn(nbytes // 4, device="cuda")
out = [torch.empty_like(src) for _ in range(m)]
for _ in range(5):
    for r, c in enumerate(comms):
        c.broadcast(src if r == 0 else None, out[r], root=0)
torch.cuda.synchronize()
tr = comms[0].trace()
t0 = min(t[0] for t in tr)
for i, t in enumerate(tr):
    print(f"cta {i}: " + " ".join(f"{(x - t0) / 1e3:6.2f}" if x else "     -" for x in t[:13]))
