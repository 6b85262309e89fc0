#!/usr/bin/env python
"""Small-size latency of the packed DGX-1V plans vs a single minimum-depth
(BFS) tree: the BFS tree is planned by giving the library a graph that holds
only the tree's links.  Device time per call (graph of 10 calls)."""
import os
import sys
from collections import deque

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402
from scripts.ab_env import per_call_us  # noqa: E402


def bfs_pairs(n, cap, root):
    par = {root: -1}
    q = deque([root])
    while q:
        u = q.popleft()
        for v in range(n):
            if v not in par and cap.get((u, v), 0) > 0:
                par[v] = u
                q.append(v)
    out = {}
    for v, u in par.items():
        if u >= 0:
            out[(u, v)] = 1
            out[(v, u)] = 1
    return out


def main():
    n, cap = OG.dgx1v()
    full = B.init_all([0] * n, graph=B.Graph.from_pairs(n, cap))
    # AllReduce centre: rank 0 (eccentricity 2 like every DGX-1V GPU)
    bfs = B.init_all([0] * n, graph=B.Graph.from_pairs(n, bfs_pairs(n, cap, 0)))
    for coll in ("bc", "ar"):
        for nbytes in (1 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20):
            xs = [torch.randn(nbytes // 4, device="cuda") for _ in range(n)]
            ys = [torch.empty_like(x) for x in xs]
            res = []
            for comms in (full, bfs):
                def fn():
                    for r, c in enumerate(comms):
                        if coll == "ar":
                            c.allreduce(xs[r], ys[r])
                        else:
                            c.broadcast(xs[0] if r == 0 else None, ys[r], root=0)
                res.append(per_call_us(fn, 10))
            print(f"{coll} {nbytes >> 10}K packed {res[0]:.1f} us  bfs {res[1]:.1f} us", flush=True)


if __name__ == "__main__":
    main()
