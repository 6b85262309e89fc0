"""Link-graph model and presets.  TEST INFRASTRUCTURE ONLY (see oracle/__init__).

P:338 (Sec. 3.1): "every GPU is a vertex V and every link (NVLink or PCIe) is
marked as a directed edge E.  Each directed edge also has a bandwidth
proportional capacity."

A graph here is ``(n, cap)`` with ``cap`` a dict ``{(u, v): c_uv}`` over
directed GPU pairs, ``c_uv`` = number of parallel links (link units, R#5:
integer capacities are what the ILP's {0,1} weights need).  A physical
bidirectional link contributes one unit in each direction.
"""
from itertools import combinations

# Fig. dgx1-topo is a [FIGURE] placeholder; the edge lists below are
# the reconstruction of SURVEY.md App. B (R#17).  They are pinned by the text's
# consequences in tests/test_oracle_graphs.py: "lack of NVLink between GPUs 1
# and 4", the 6-GPU unused links {1-3, 5-7, 0-4}, the ring
# 2-6-7-3-2, 46/14 topology-unique allocations, and the
# 6 unit-rate trees of DGX-1V.
DGX1P_PAIRS = [(0, 1), (0, 2), (0, 3), (0, 4), (1, 2), (1, 3), (1, 5), (2, 3),
               (2, 6), (3, 7), (4, 5), (4, 6), (4, 7), (5, 6), (5, 7), (6, 7)]
# "red dashed-lines are the additional NVLinks in DGX-1-V100 servers":
# the V100 has 6 NVLink ports, so 8 of the 16 P100 pairs are doubled.
DGX1V_DOUBLED = [(0, 3), (0, 4), (1, 2), (1, 5), (2, 3), (4, 7), (5, 6), (6, 7)]


def from_pairs(n, pairs, mult=None):
    """Undirected pair list -> directed capacity dict (one unit per direction
    per parallel link, SPEC-style bidirectional expansion)."""
    cap = {}
    for (u, v) in pairs:
        k = 1 if mult is None else mult.get((min(u, v), max(u, v)), 1)
        cap[(u, v)] = cap.get((u, v), 0) + k
        cap[(v, u)] = cap.get((v, u), 0) + k
    return n, cap


def dgx1p():
    """DGX-1P (P100, NVLink gen1): 16 links, 4 per GPU."""
    return from_pairs(8, DGX1P_PAIRS)


def dgx1v():
    """DGX-1V (V100, NVLink gen2): the P100 pairs plus 8 doubled pairs, 6 per GPU."""
    mult = {p: 2 for p in DGX1V_DOUBLED}
    return from_pairs(8, DGX1P_PAIRS, mult)


def complete(m, c=1):
    """K_m with capacity c per directed pair (the NVSwitch model, R#10)."""
    return m, {(u, v): c for u in range(m) for v in range(m) if u != v}


def induced(g, nodes):
    """Induced sub-allocation ("infer the interconnect topology across
    only the GPUs allocated"), relabelled to 0..k-1 in ascending order of the
    original ids.  Returns (graph, original_ids)."""
    n, cap = g
    ids = sorted(nodes)
    idx = {v: i for i, v in enumerate(ids)}
    sub = {(idx[u], idx[v]): c for (u, v), c in cap.items() if u in idx and v in idx}
    return (len(ids), sub), ids


def undirected_pairs(g):
    """{(u,v) u<v: capacity} -- AllReduce's undirected model.  The
    capacity of an undirected link is its per-direction capacity (R#9)."""
    n, cap = g
    out = {}
    for (u, v), c in cap.items():
        a, b = min(u, v), max(u, v)
        if (v, u) not in cap:
            raise ValueError(f"link {u}->{v} has no reverse edge (AllReduce needs bidirectional links, P:397)")
        out[(a, b)] = min(c, cap[(v, u)])
    return out


def is_connected(g):
    n, cap = g
    if n <= 1:
        return True
    adj = {u: set() for u in range(n)}
    for (u, v) in cap:
        adj[u].add(v)
        adj[v].add(u)
    seen, stack = {0}, [0]
    while stack:
        u = stack.pop()
        for w in adj[u]:
            if w not in seen:
                seen.add(w)
                stack.append(w)
    return len(seen) == n


def canonical_form(g):
    """Brute-force canonical form of a small multigraph: the lexicographically
    smallest sorted edge-multiset over all relabellings.  Used to bin
    allocations "by topology uniqueness"."""
    from itertools import permutations
    n, cap = g
    best = None
    for perm in permutations(range(n)):
        key = tuple(sorted((perm[u], perm[v], c) for (u, v), c in cap.items()))
        if best is None or key < best:
            best = key
    return (n, best)


def unique_allocations(g, sizes=range(3, 9)):
    """Number of distinct (isomorphism classes of) connected induced
    sub-allocations for each size k."""
    n, _ = g
    out = {}
    for k in sizes:
        forms = set()
        for nodes in combinations(range(n), k):
            sub, _ = induced(g, nodes)
            if is_connected(sub):
                forms.add(canonical_form(sub))
        out[k] = len(forms)
    return out
