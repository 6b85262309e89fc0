#!/usr/bin/env python
"""MIAD (NEXT-2) trajectories on the GPU: chunk size and measured
throughput per call for configs where chunking matters.  Writes JSON."""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402  (topology preset only)


def trace(comms, coll, S, iters=16):
    m = len(comms)
    cnt = S // 4
    xs = [torch.randn(cnt, device="cuda") for _ in range(m)]
    ys = [torch.empty_like(x) for x in xs]
    rows = []
    for it in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r, c in enumerate(comms):
            if coll == "allreduce":
                c.allreduce(xs[r], ys[r])
            else:
                c.broadcast(xs[0] if r == 0 else None, ys[r], root=0)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        st = comms[0].stats()
        rows.append({"iter": it, "chunk_bytes": st["last_chunk_bytes"], "ctas": st["last_ctas"],
                     "ms": round(ms, 4), "algbw": round(S / ms / 1e6, 1)})
    return rows


def main():
    out = {}
    g = OG.dgx1v()
    comms = B.init_all([0] * 8, graph=B.Graph.from_pairs(8, g[1]), cfg=B.config(autotune=1))
    out["c2-dgx1v-broadcast-256MiB"] = trace(comms, "broadcast", 256 << 20)
    for c in comms:
        c.destroy()
    comms = B.init_all([0] * 8, cfg=B.config(autotune=1))
    out["c3-onehop-allreduce-64MiB"] = trace(comms, "allreduce", 64 << 20)
    for c in comms:
        c.destroy()
    tri, _ = OG.induced(OG.dgx1p(), [0, 1, 3])
    comms = B.init_all([0] * 3, graph=B.Graph.from_pairs(3, tri[1]), cfg=B.config(autotune=1))
    out["c1-3gpu-broadcast-64MiB"] = trace(comms, "broadcast", 64 << 20)
    for k, rows in out.items():
        print(k)
        for r in rows:
            print("  ", r)
    path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "miad_trace.json")
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
