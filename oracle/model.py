"""Timing and traffic models of chunked tree collectives (oracle; TEST
INFRASTRUCTURE ONLY -- see oracle/__init__.py).

pipeline_makespan  discrete-event simulation of chunk forwarding along a
                   tree (Sec. 4.2 "Automatic chunk size selection",
                   Fig. chunk-data): a node forwards a chunk only once it has
                   received all of it; each directed link carries one chunk at
                   a time; every link moves the whole buffer in `t_link`.
chain_time         the closed form for a chain of h hops and c equal chunks,
                   (c + h - 1) / c * t_link (SURVEY 8(c-5) "Pipeline").
link_bytes         bytes carried per directed link by a plan for a buffer of S
                   bytes, split by weight (R#11): Broadcast moves tree
                   i's range once along every edge (root -> leaves); AllReduce
                   moves it once up (reduce) and once down (broadcast) along
                   every edge.
"""
from fractions import Fraction

from . import packing


def pipeline_makespan(parent, nchunks, t_link=Fraction(1)):
    """Finish time of a chunked Broadcast of one buffer along the tree
    `parent` (parent[root] = -1) when the buffer is cut into `nchunks` equal
    chunks.  Events are simulated chunk by chunk in order: chunk c can leave
    node u for child v once u holds all of chunk c and link (u, v) has
    finished chunk c - 1.  Returns the time the last node holds the last
    chunk (exact Fraction)."""
    n = len(parent)
    root = parent.index(-1)
    kids = {u: [v for v in range(n) if parent[v] == u] for u in range(n)}
    per_chunk = Fraction(t_link) / nchunks
    have = {root: [Fraction(0)] * nchunks}   # have[u][c]: time u holds chunk c
    link_free = {}
    order = [root]
    for u in order:                          # BFS: parents before children
        for v in kids[u]:
            order.append(v)
            times = []
            for c in range(nchunks):
                start = max(have[u][c], link_free.get((u, v), Fraction(0)))
                done = start + per_chunk
                link_free[(u, v)] = done
                times.append(done)
            have[v] = times
    return max(t[-1] for t in have.values())


def chain_time(nchunks, hops, t_link=Fraction(1)):
    """(c + h - 1) / c * t_link: the pipelined time of c chunks over h hops."""
    return Fraction(nchunks + hops - 1, nchunks) * t_link


def link_bytes(plan, n, S, allreduce):
    """{(u, v): bytes} on every directed link used by `plan` for S bytes per
    rank.  Tree i carries its exact split range (packing.split_bytes)."""
    ranges = packing.split_bytes(S, [t["weight"] for t in plan["trees"]])
    out = {}
    for t, (lo, hi) in zip(plan["trees"], ranges):
        b = hi - lo
        for v, p in enumerate(t["parent"]):
            if p < 0:
                continue
            out[(p, v)] = out.get((p, v), 0) + b          # broadcast direction
            if allreduce:
                out[(v, p)] = out.get((v, p), 0) + b      # reduce direction
    return out


def hybrid_split(d_total, bw_pcie, bw_nvl, t_dpa):
    """Eq. 8 (Sec. 3.4 "Handling hybrid communication"): split
    D_total between the PCIe trees and the NVLink trees so that
    T_PCIe + T_dpa = T_NVL, i.e.
        D_PCIe = D_total * BW_PCIe / (BW_PCIe + BW_NVL)
                 - T_dpa * BW_PCIe * BW_NVL / (BW_PCIe + BW_NVL),
        D_NVL  = D_total - D_PCIe.
    The paper leaves the infeasible case silent; R#31: D_PCIe is clamped to
    [0, D_total] (a large T_dpa sends everything over NVLink).  Exact
    rationals in, exact rationals out."""
    d_total, bw_pcie, bw_nvl, t_dpa = (Fraction(x) for x in (d_total, bw_pcie, bw_nvl, t_dpa))
    d_pcie = d_total * bw_pcie / (bw_pcie + bw_nvl) - t_dpa * bw_pcie * bw_nvl / (bw_pcie + bw_nvl)
    d_pcie = min(max(d_pcie, Fraction(0)), d_total)
    return d_pcie, d_total - d_pcie
