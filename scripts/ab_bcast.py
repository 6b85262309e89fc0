#!/usr/bin/env python
"""A/B helper: per-call device time (graph of 10 calls) of the multi-hop
Broadcast configs (c1 triangle chains, c2 DGX-1V packed trees, c3 switch
two-level trees) and the DGX-1V multi-level AllReduce over sizes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402
from scripts.ab_env import per_call_us  # noqa: E402

SIZES = (1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20)


def main():
    tri, _ = OG.induced(OG.dgx1p(), [0, 1, 3])
    cfgs = [("c1", 3, B.Graph.from_pairs(3, tri[1]), "bc"), ("c2", 8, B.Graph.from_pairs(8, OG.dgx1v()[1]), "bc"),
            ("c3", 8, None, "bc"), ("c2ar", 8, B.Graph.from_pairs(8, OG.dgx1v()[1]), "ar")]
    for name, m, G, coll in cfgs:
        comms = B.init_all([0] * m, graph=G)
        out = []
        for nbytes in SIZES:
            xs = [torch.randn(nbytes // 4, device="cuda") for _ in range(m)]
            ys = [torch.empty_like(x) for x in xs]

            def fn():
                for r, c in enumerate(comms):
                    if coll == "ar":
                        c.allreduce(xs[r], ys[r])
                    else:
                        c.broadcast(xs[0] if r == 0 else None, ys[r], root=0)
            us = per_call_us(fn, 10 if nbytes <= (16 << 20) else 3, per_graph=5)
            out.append(f"{nbytes >> 20}M:{us:.1f}")
            del xs, ys
        print(f"{os.environ.get('CFG_LABEL', '')} {name} " + " ".join(out), flush=True)
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
