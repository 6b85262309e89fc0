"""Optimal packing rates: closed-form bounds and brute-force LPs.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Eqs. 1-3 (Sec. 3.1): max sum_i w_i  s.t. for all e:
sum_i kappa_{i,e} w_i <= c_e, kappa_{i,e} = [e in T_i]  (R#1: "<" read as
"<="; R#2: kappa carries the edge index).

Edmonds / Lovasz (cited P:195): the optimum over *all* arborescences
rooted at r equals min_{v != r} maxflow(r -> v).

For AllReduce's undirected model the optimum fractional packing of
spanning trees is the Nash-Williams/Tutte partition bound
min_P cross(P) / (|P| - 1).

The brute-force LP enumerates every tree (feasible up to 8 nodes: <= 16384
parent assignments), so it pins both bounds independently.
"""
from collections import deque
from itertools import product

import numpy as np


def maxflow(n, cap, s, t):
    """Edmonds-Karp on a capacity dict {(u,v): c}.  Plain BFS augmenting paths."""
    res = {}
    for (u, v), c in cap.items():
        res[(u, v)] = res.get((u, v), 0) + c
        res.setdefault((v, u), 0)
    adj = {u: [] for u in range(n)}
    for (u, v) in res:
        adj[u].append(v)
    flow = 0
    while True:
        prev = {s: None}
        q = deque([s])
        while q and t not in prev:
            u = q.popleft()
            for v in adj[u]:
                if v not in prev and res[(u, v)] > 0:
                    prev[v] = u
                    q.append(v)
        if t not in prev:
            return flow
        # bottleneck
        b, v = float("inf"), t
        while prev[v] is not None:
            b = min(b, res[(prev[v], v)])
            v = prev[v]
        v = t
        while prev[v] is not None:
            u = prev[v]
            res[(u, v)] -= b
            res[(v, u)] += b
            v = u
        flow += b


def edmonds_rate(g, r):
    """Optimal broadcast rate from r: min over v != r of maxflow(r -> v)."""
    n, cap = g
    return min(maxflow(n, cap, r, v) for v in range(n) if v != r)


def enumerate_arborescences(g, r):
    """Every arborescence rooted at r, as a parent tuple (parent[r] = -1).
    Brute force: each non-root vertex picks one in-neighbour; keep the choices
    in which every vertex reaches r without a cycle."""
    n, cap = g
    choices = []
    for v in range(n):
        if v == r:
            choices.append([-1])
        else:
            choices.append(sorted({u for (u, w) in cap if w == v}))
    out = []
    for parent in product(*choices):
        ok = True
        for v in range(n):
            seen, x = set(), v
            while x != r:
                if x in seen:
                    ok = False
                    break
                seen.add(x)
                x = parent[x]
            if not ok:
                break
        if ok:
            out.append(tuple(parent))
    return out


def arborescence_edges(parent):
    return [(p, v) for v, p in enumerate(parent) if p >= 0]


def enumerate_spanning_trees(pairs, n):
    """Every undirected spanning tree over `pairs` ({(u,v) u<v: c}), as a sorted
    tuple of (u,v) pairs.  Each undirected spanning tree is exactly one
    arborescence rooted at 0 of the symmetric digraph."""
    sym = {}
    for (u, v), c in pairs.items():
        sym[(u, v)] = c
        sym[(v, u)] = c
    trees = set()
    for parent in enumerate_arborescences((n, sym), 0):
        trees.add(tuple(sorted((min(p, v), max(p, v)) for (p, v) in arborescence_edges(parent))))
    return sorted(trees)


def packing_lp(edge_caps, trees_edges):
    """max sum w  s.t.  sum_{T contains e} w_T <= c_e, w >= 0   (Eqs. 1-3).
    `trees_edges`: list of edge lists.  Returns (rate, weights).  scipy's HiGHS
    LP is the library primitive."""
    from scipy.optimize import linprog
    edges = sorted(edge_caps)
    eidx = {e: i for i, e in enumerate(edges)}
    A = np.zeros((len(edges), len(trees_edges)))
    for j, te in enumerate(trees_edges):
        for e in te:
            A[eidx[e], j] += 1.0
    b = np.array([edge_caps[e] for e in edges], dtype=float)
    res = linprog(-np.ones(len(trees_edges)), A_ub=A, b_ub=b, bounds=(0, None), method="highs")
    assert res.status == 0, res.message
    return -res.fun, res.x


def brute_broadcast_rate(g, r):
    """Exact optimum of Eqs. 1-3 over every arborescence rooted at r."""
    n, cap = g
    trees = [arborescence_edges(p) for p in enumerate_arborescences(g, r)]
    return packing_lp(cap, trees)[0]


def brute_allreduce_rate(pairs, n):
    """Exact optimum of the undirected packing LP over every spanning tree."""
    trees = enumerate_spanning_trees(pairs, n)
    return packing_lp(pairs, [list(t) for t in trees])[0]


def set_partitions(items):
    """All set partitions of a list (Bell-number many; 4140 for 8 items)."""
    if not items:
        yield []
        return
    first, rest = items[0], items[1:]
    for part in set_partitions(rest):
        for i in range(len(part)):
            yield part[:i] + [[first] + part[i]] + part[i + 1:]
        yield [[first]] + part


def nash_williams_rate(pairs, n):
    """min over partitions P (|P| >= 2) of cross(P) / (|P| - 1)."""
    best = float("inf")
    for part in set_partitions(list(range(n))):
        if len(part) < 2:
            continue
        block = {}
        for i, b in enumerate(part):
            for v in b:
                block[v] = i
        cross = sum(c for (u, v), c in pairs.items() if block[u] != block[v])
        best = min(best, cross / (len(part) - 1))
    return best
