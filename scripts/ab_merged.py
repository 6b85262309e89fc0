#!/usr/bin/env python
"""Merged one-hop AllReduce (switch, m virtual ranks, one launch) over small and
medium sizes, f32 and bf16: per-call device time.  CFG_LABEL=x python scripts/ab_merged.py"""
import os
import sys

sys.path.insert(0, os.environ.get("AB_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1910_04940_b200 as B  # noqa: E402
from sweep import run_coll  # noqa: E402

label = os.environ.get("CFG_LABEL", "")
for m in (8, 5, 3, 2):
    comms = B.init_all([0] * m)
    for dt in ("f32", "bf16"):
        parts = []
        for kb in (256, 1024, 2048, 4096, 6144, 8192):
            r = run_coll(comms, "allreduce", kb << 10, dt, 0, "x")
            parts.append(f"{kb >> 10 if kb >= 1024 else kb}{'M' if kb >= 1024 else 'K'}:{r['ms'] * 1e3:.1f}")
        print(f"{label:8s} m={m} {dt:4s} " + " ".join(parts), flush=True)
    for c in comms:
        c.destroy()
