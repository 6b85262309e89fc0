#!/usr/bin/env python
"""Batched single launch vs per-rank launches (cfg.launch_per_rank) on one B200.

    python scripts/per_rank_sweep.py [--out profiles/per_rank_sweep_rNN.json] [--max-mib 256]

Per-rank launches run the one-process-per-GPU protocol (entry handshake,
per-chunk flags across launches, exit waits) concurrently on one GPU, each
rank's launch with 1/m of the SMs.  The difference to the batched launch is
the protocol's cost.  Rows as in scripts/sweep.py (CUDA-graph replay device
time per call) plus "mode".
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402  (topology presets only)
from sweep import run_coll, sizes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--max-mib", type=int, default=256)
    ap.add_argument("--step", type=int, default=4)
    args = ap.parse_args()
    hi = args.max_mib << 20
    rows = []
    for mode, per_rank in (("batched", 0), ("per_rank", 1)):
        cfg = B.config(launch_per_rank=per_rank, timeout_s=30.0)
        comms = B.init_all([0] * 8, cfg=cfg)
        for S in sizes(1 << 10, hi, args.step):
            for coll in ("allreduce", "broadcast"):
                r = run_coll(comms, coll, S, "f32", 0, "c3-switch")
                r["mode"] = mode
                rows.append(r)
                print(json.dumps(r), flush=True)
        for c in comms:
            c.destroy()
        g = OG.dgx1v()
        comms = B.init_all([0] * 8, graph=B.Graph.from_pairs(8, g[1]), cfg=cfg)
        for S in sizes(1 << 10, hi, args.step * 4):
            r = run_coll(comms, "broadcast", S, "f32", 0, "c2-dgx1v-emulated")
            r["mode"] = mode
            rows.append(r)
            print(json.dumps(r), flush=True)
        for c in comms:
            c.destroy()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"rows": rows}, f, indent=0)


if __name__ == "__main__":
    main()
