#!/usr/bin/env python
"""A/B of small and medium calls on the switch (virtual ranks, m = 8): one-hop
AllReduce (merged launch / LL), Broadcast, ReduceScatter / AllGather; device
time per call (scripts/sweep.py timing).  CFG_LABEL=x [AB_ROOT=...] python scripts/ab_small.py"""
import os
import sys

sys.path.insert(0, os.environ.get("AB_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1910_04940_b200 as B  # noqa: E402
from sweep import run_block, run_coll  # noqa: E402

label = os.environ.get("CFG_LABEL", "")
comms = B.init_all([0] * 8)
for coll in ("allreduce", "broadcast"):
    parts = [f"{S >> 10}K:{run_coll(comms, coll, S, 'f32', 0, 'x')['ms'] * 1e3:.1f}"
             for S in (1 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20)]
    print(f"{label:8s} {coll:15s} " + " ".join(parts), flush=True)
for coll in ("reduce_scatter", "allgather"):
    parts = [f"{S >> 10}K:{run_block(comms, coll, S, 'f32', 'x')['ms'] * 1e3:.1f}"
             for S in (64 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20)]
    print(f"{label:8s} {coll:15s} " + " ".join(parts), flush=True)
