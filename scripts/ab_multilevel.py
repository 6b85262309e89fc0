#!/usr/bin/env python
"""A/B of the multi-hop configurations (virtual ranks): per-call device time
(scripts/sweep.py's timing) of every plan with deep or multi-level trees.

    CFG_LABEL=x [BLINK_...=...] python scripts/ab_multilevel.py [sizes MiB, default 1,16,64,256]

One line per (config, collective): label, then size:us pairs and plan_hbm_frac.
"""
import os
import sys

sys.path.insert(0, os.environ.get("AB_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402  (topology presets only)
from sweep import run_coll  # noqa: E402

SIZES = [int(float(x) * (1 << 20)) for x in (sys.argv[1].split(",") if len(sys.argv) > 1 else "1,16,64,256".split(","))]
ONLY = os.environ.get("AB_ONLY", "")
label = os.environ.get("CFG_LABEL", "")


def case(tag, comms, colls):
    if ONLY and ONLY not in tag:
        for c in comms:
            c.destroy()
        return
    for coll in colls:
        parts = []
        for S in SIZES:
            r = run_coll(comms, coll, S, "f32", 0, tag)
            parts.append(f"{S / (1 << 20):g}M:{r['ms'] * 1e3:.1f}us/{r['plan_hbm_frac']:.2f}")
        print(f"{label:10s} {tag:22s} {coll:9s} " + " ".join(parts), flush=True)
    for c in comms:
        c.destroy()


g = OG.dgx1v()
tri, _ = OG.induced(OG.dgx1p(), [0, 1, 3])
case("c1-3gpu", B.init_all([0] * 3, graph=B.Graph.from_pairs(3, tri[1])), ["broadcast"])
case("c2-dgx1v", B.init_all([0] * 8, graph=B.Graph.from_pairs(8, g[1])), ["broadcast", "allreduce"])
case("c3-switch", B.init_all([0] * 8), ["broadcast"])
for nodes in ([0, 1, 3, 4, 5, 7], [1, 4, 5, 6]):
    sub, _ = OG.induced(g, nodes)
    case(f"c4-dgx1v-{''.join(map(str, nodes))}",
         B.init_all([0] * len(nodes), graph=B.Graph.from_pairs(len(nodes), sub[1])), ["allreduce"])
for servers in ([[0, 1, 3], [2, 4, 5, 6, 7]], [[0, 1, 2, 3], [4, 5, 6, 7]]):
    case("next4-" + "+".join(str(len(s)) for s in servers),
         B.init_all([0] * 8, graph=B.Graph.multi_server(8, g[1], servers)), ["allreduce"])
