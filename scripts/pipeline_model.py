#!/usr/bin/env python
"""Chunk pipelining on the B200 vs the paper's model ("two chunks
save a third", t = (c + h - 1) / c * T for c chunks over h hops).

Broadcast of S bytes down a path 0 -> 1 -> ... -> 7 (one tree, h = 7 hops)
with the chunk size fixed to S / c (cfg.chunk_bytes), c = 1 .. 128.  A chunk
is the unit of work of one CTA, and each hop's channel has k CTAs taking
chunks in order, so a hop moves up to k chunks at once: the paper's model
with k chunks in flight per hop,
    T(c) = (ceil(c / k) + h - 1) * (S / (c * b) + lam)
(b = one CTA's copy bandwidth, lam = per-chunk per-hop overhead: flag
signal, store drain, poll), is fitted to the per-call device time (graph of
5 calls) by least squares; the JSON records every point, the fit and its
residuals.  With k = 1 it is exactly P:510-513's (c + h - 1) / c.

    python scripts/pipeline_model.py [--out profiles/pipeline_r01.json]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
from scripts.ab_env import per_call_us  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    m = 8
    h = m - 1
    G = B.Graph(m, [(v, v + 1, 1.0, 1) for v in range(m - 1)])
    rows = []
    for S in (4 << 20, 16 << 20, 64 << 20):
        x = torch.randn(S // 4, device="cuda")
        ys = [torch.empty_like(x) for _ in range(m)]
        for c in (1, 2, 4, 8, 16, 32, 64, 128):
            chunk = S // c
            comms = B.init_all([0] * m, graph=G, cfg=B.config(chunk_bytes=chunk))
            p = comms[0].plan(False, 0, S // 4)
            assert len(p["trees"]) == 1 and p["trees"][0]["depth"] == h and p["trees"][0]["nchunks"] == c

            def fn():
                for r, cm in enumerate(comms):
                    cm.broadcast(x if r == 0 else None, ys[r], root=0)
            us = per_call_us(fn, 5, per_graph=5)
            torch.cuda.synchronize()
            for y in ys[1:]:
                assert torch.equal(y, x)
            k = comms[0].stats()["last_ctas"] / h  # CTAs per hop channel (the leaf has none)
            rows.append({"S": S, "chunks": c, "chunk_bytes": chunk, "us": round(us, 2), "ctas_per_hop": k})
            print(rows[-1], flush=True)
            for cm in comms:
                cm.destroy()
    # least squares per S: T = (ceil(c/k)+h-1) * (S/(c b) + lam), linear in (1/b, lam)
    fits = []
    for S in sorted({r["S"] for r in rows}):
        pts = [r for r in rows if r["S"] == S]
        w = [np.ceil(r["chunks"] / r["ctas_per_hop"]) + h - 1 for r in pts]
        A = np.array([[wi * S / r["chunks"], wi] for wi, r in zip(w, pts)])
        t = np.array([r["us"] * 1e-6 for r in pts])
        (inv_b, lam), *_ = np.linalg.lstsq(A, t, rcond=None)
        pred = A @ np.array([inv_b, lam])
        best = min(pts, key=lambda r: r["us"])
        fits.append({"S": S, "b_GBps_per_cta": round(float(1 / inv_b / 1e9), 1), "lam_us": round(float(lam * 1e6), 2),
                     "max_rel_residual": round(float(np.max(np.abs(pred - t) / t)), 3),
                     "best_chunks": best["chunks"], "best_us": best["us"],
                     "unpipelined_us": [r["us"] for r in pts if r["chunks"] == 1][0],
                     "speedup_best_vs_unpipelined": round([r["us"] for r in pts if r["chunks"] == 1][0] / best["us"], 2),
                     "ctas_per_hop": pts[0]["ctas_per_hop"],
                     "pred_us": [round(float(x) * 1e6, 1) for x in pred]})
        print(fits[-1], flush=True)
    out = {"graph": "path 0-1-...-7 (h = 7 hops), Broadcast from 0, virtual ranks on one B200",
           "model": "T(c) = (ceil(c/k) + h - 1) * (S / (c b) + lam); k = 1 is P:510-513's (c + h - 1) / c",
           "rows": rows, "fits": fits}
    if args.out:
        json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
