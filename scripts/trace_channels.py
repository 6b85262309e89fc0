#!/usr/bin/env python
"""BLINK_TRACE + BLINK_DEBUG_TASKS on one call: per channel (rank, tree,
role, parent, children) the CTA count, first-load and last-store times (us).

    python scripts/trace_channels.py <graph: dgx1v|dgx1v:<ids>|switch:<m>> <ar|bc> <bytes>
"""
import os
import re
import subprocess
import sys

if os.environ.get("_TC_CHILD") != "1":
    env = dict(os.environ, _TC_CHILD="1", BLINK_TRACE="1", BLINK_DEBUG_TASKS="1")
    r = subprocess.run([sys.executable] + sys.argv, env=env, capture_output=True, text=True)
    tasks = {}
    for l in r.stderr.splitlines():
        m = re.match(r"\[blink\] cta (\d+) rank (\d+) tree (\d+) role (\d+) parent (-?\d+) children (\w+) chunks (\d+)", l)
        if m:
            tasks[int(m[1])] = (int(m[2]), int(m[3]), int(m[4]), int(m[5]), m[6], int(m[7]))
        elif "alloc:" in l:
            print(l)
    ct = {}
    for l in r.stdout.splitlines():
        m = re.match(r"cta (\d+): (.*)", l)
        if m:
            ct[int(m[1])] = [float(x) if x != "-" else None for x in m[2].split()]
        elif l.strip():
            print(l)
    ch = {}
    for i, v in ct.items():
        ch.setdefault(tasks.get(i), []).append(v)
    rows = []
    for k, v in ch.items():
        ends = [x[5] for x in v if x[5] is not None]
        firsts = [x[3] for x in v if x[3] is not None]
        rows.append((max(ends) if ends else 0, min(firsts) if firsts else 0, len(v), k))
    for e, f, n, k in sorted(rows):
        print(f"end {e:8.1f} first {f:7.1f} ctas {n:3d} (rank, tree, role, parent, children, chunks) = {k}")
    sys.exit(r.returncode)

import torch  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
from oracle import graphs as OG  # noqa: E402

gspec, coll, S = sys.argv[1], sys.argv[2], int(sys.argv[3])
if gspec.startswith("switch"):
    m = int(gspec.split(":")[1])
    comms = B.init_all([0] * m)
else:
    g = OG.dgx1v()
    if ":" in gspec:
        ids = [int(c) for c in gspec.split(":")[1]]
        g, _ = OG.induced(g, ids)
    m = g[0]
    comms = B.init_all([0] * m, graph=B.Graph.from_pairs(m, g[1]))
cnt = S // 4
xs = [torch.randn(cnt, device="cuda") for _ in range(m)]
ys = [torch.empty_like(x) for x in xs]
for _ in range(3):
    for r, c in enumerate(comms):
        if coll == "ar":
            c.allreduce(xs[r], ys[r])
        else:
            c.broadcast(xs[0] if r == 0 else None, ys[r], root=0)
torch.cuda.synchronize()
tr = comms[0].trace()
t0 = min(t[0] for t in tr)
print("kernel end", max((t[7] - t0) / 1e3 for t in tr), "us")
for i, t in enumerate(tr):
    print(f"cta {i}: " + " ".join(f"{(x - t0) / 1e3:.1f}" if x else "-" for x in t[:8]))
