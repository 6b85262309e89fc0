#!/usr/bin/env python
"""A few identical calls of one collective (for ncu captures):
    python scripts/one_call.py M BYTES DTYPE [ar|bc] [calls]
ONE_CALL_GRAPH=dgx1v plans on the emulated DGX-1V link graph (M = 8)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402

m, nbytes = int(sys.argv[1]), int(sys.argv[2])
dt = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32}[sys.argv[3]]
coll = sys.argv[4] if len(sys.argv) > 4 else "ar"
calls = int(sys.argv[5]) if len(sys.argv) > 5 else 3
graph = None
if os.environ.get("ONE_CALL_GRAPH") == "dgx1v":
    from oracle import graphs as OG  # topology preset only
    graph = B.Graph.from_pairs(8, OG.dgx1v()[1])
comms = B.init_all([0] * m, graph=graph)
es = torch.empty((), dtype=dt).element_size()
xs = [torch.randn(nbytes // es, device="cuda").to(dt) for _ in range(m)]
ys = [torch.empty_like(x) for x in xs]
for _ in range(calls):
    for r, c in enumerate(comms):
        if coll == "ar":
            c.allreduce(xs[r], ys[r])
        else:
            c.broadcast(xs[0] if r == 0 else None, ys[r], root=0)
torch.cuda.synchronize()
print("ok")
