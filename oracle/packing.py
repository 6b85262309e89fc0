"""Tree packing: MWU, ILP refinement, one-hop switch trees, weight split.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Follows the paper step by step:

* Sec. 3.2: "at each iteration we find the minimum weight spanning
  tree given the current assignment.  We then increment the weight on this
  chosen tree by an epsilon factor and update weights on the graph
  correspondingly."  Step rule (R#4): Garg-Koenemann with bottleneck routing,
  lengths l_e = delta / c_e kept as logs and normalised by their max before
  each minimum-tree call (without normalisation the raw lengths
  ~1e-34 lose the (1 - eps) guarantee).  Final uniform scaling to exact
  feasibility; identical trees merged.
* Sec. 3.2.1 (Eqs. 4-7): binary ILP over the MWU candidates ("k
  here is controlled by the number of trees returned by the MWU procedure",
  P:390; the candidates are the trees of four MWU runs, R#21), then
  "iteratively relax the constraints (i.e. allowing w_i to take fractional
  values) until c_hat is within a configured threshold (e.g., 5%) of c*"
  (R#5, R#6: grid w in {0, 1/g, ..., 1} for g = 1, 2, 4, 8, 16; gap 0.05;
  R#3: c* = the optimal rate, exact where computable).  No other candidates
  and no weight above 1 (Eq. 6): the product's extra heuristics (R#21, R#26)
  are not part of the oracle.
* Sec. 3.3: AllReduce packs *undirected* spanning trees (a tree
  of weight w consumes w on the link in both directions); the per-tree root is
  the tree's centre (R#9).
* Sec. 3.5: on a switch, m one-hop trees, each GPU root of 1/m.
* Sec. 4.1: "split the buffer among all the spanning trees based on
  their weights" -- 16-byte-grain prefix-floor split (R#11).
"""
import math
from fractions import Fraction

import numpy as np

GRAIN = 16  # bytes; R#11


# --------------------------------------------------------------------------
# Minimum-weight arborescence (Chu-Liu / Edmonds), the MWU inner oracle
# --------------------------------------------------------------------------
def _tie_key(e, tiebreak):
    """Deterministic tie-break among equal lengths: lexicographic
    (src, dst) ascending ("asc") or descending ("desc", the alternate run of
    SURVEY 7 hard part 8)."""
    return e if tiebreak == "asc" else (-e[0], -e[1])


def min_arborescence(n, r, lengths, tiebreak="asc"):
    """Minimum-total-length arborescence rooted at r.

    `lengths`: {(u, v): l}.  Ties: smallest (length, tie key) in-edge.
    Returns a parent tuple (parent[r] = -1).  Plain recursive contraction."""
    edges = [(u, v, w, _tie_key((u, v), tiebreak)) for (u, v), w in lengths.items() if u != v]
    chosen = _cle(n, r, edges)
    parent = [-1] * n
    for key in chosen:
        u, v = key if tiebreak == "asc" else (-key[0], -key[1])
        parent[v] = u
    return tuple(parent)


def _cle(n, r, edges):
    # 1. cheapest incoming edge per non-root vertex
    inb = {}
    for e in edges:
        u, v, w, key = e
        if v == r or u == v:
            continue
        if v not in inb or (w, key) < (inb[v][2], inb[v][3]):
            inb[v] = e
    for v in range(n):
        if v != r and v not in inb:
            raise ValueError(f"vertex {v} unreachable from root {r}")
    # 2. cycles among the chosen edges
    comp = [-1] * n
    mark = [-1] * n
    ncomp = 0
    cyclic = False
    for v in range(n):
        x = v
        while x != r and mark[x] == -1 and comp[x] == -1:
            mark[x] = v
            x = inb[x][0]
        if x != r and mark[x] == v and comp[x] == -1:
            # x lies on a new cycle
            cyclic = True
            y = x
            while True:
                comp[y] = ncomp
                y = inb[y][0]
                if y == x:
                    break
            ncomp += 1
    if not cyclic:
        return {inb[v][3] for v in range(n) if v != r}
    for v in range(n):
        if comp[v] == -1:
            comp[v] = ncomp
            ncomp += 1
    # 3. contract and recurse; reduced cost w - w(inb[v])
    new_edges = []
    origin = {}
    for e in edges:
        u, v, w, key = e
        cu, cv = comp[u], comp[v]
        if cu == cv or v == r:
            continue
        ne = (cu, cv, w - inb[v][2], key)
        new_edges.append(ne)
        origin[key] = e
    sub = _cle(ncomp, comp[r], new_edges)
    # 4. expand: a vertex entered by a recursive choice keeps it; others keep inb
    entered = {origin[k][1]: k for k in sub}
    return {entered[v] if v in entered else inb[v][3] for v in range(n) if v != r}


def min_spanning_tree(n, lengths, tiebreak="asc"):
    """Kruskal over undirected {(u,v) u<v: l}; ties by (l, tie key of (u, v)).
    Returns a sorted tuple of (u, v) pairs."""
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    out = []
    for (w, _, (u, v)) in sorted((w, _tie_key(e, tiebreak), e) for e, w in lengths.items()):
        a, b = find(u), find(v)
        if a != b:
            parent[a] = b
            out.append((u, v))
    if len(out) != n - 1:
        raise ValueError("graph is disconnected")
    return tuple(sorted(out))


def _logsumexp(xs):
    m = max(xs)
    return m + math.log(sum(math.exp(x - m) for x in xs))


# --------------------------------------------------------------------------
# MWU (Sec. 3.2)
# --------------------------------------------------------------------------
def _mwu(caps, tree_of, eps):
    """Generic Garg-Koenemann loop over a capacity dict `caps`; `tree_of(lengths)`
    returns a tree as a hashable object and its edge list.
    Returns ({tree: weight}, c*) with weights scaled to exact feasibility."""
    edges = sorted(caps)
    mE = len(edges)
    log_delta = math.log1p(eps) - (1.0 / eps) * math.log((1.0 + eps) * mE)
    logl = {e: log_delta - math.log(caps[e]) for e in edges}
    x = {}
    tree_edges = {}
    iters = 0
    while True:
        mx = max(logl.values())
        lengths = {e: math.exp(logl[e] - mx) for e in edges}
        T, Te = tree_of(lengths)
        if _logsumexp([logl[e] for e in Te]) >= 0.0:   # sum_{e in T} l_e >= 1
            break
        cmin = min(caps[e] for e in Te)
        x[T] = x.get(T, 0.0) + cmin
        tree_edges[T] = Te
        for e in Te:
            logl[e] += math.log1p(eps * cmin / caps[e])
        iters += 1
        if iters > 10_000_000:
            raise RuntimeError("MWU did not terminate")
    load = {e: 0.0 for e in edges}
    for T, w in x.items():
        for e in tree_edges[T]:
            load[e] += w
    lam = max(load[e] / caps[e] for e in edges)
    w = {T: v / lam for T, v in x.items()}
    return w, tree_edges, sum(w.values()), iters


def mwu_broadcast(g, r, eps=0.1, tiebreak="asc"):
    """MWU packing of arborescences rooted at r on the directed graph.
    Returns (weights {parent_tuple: w}, rate c*, iterations)."""
    n, cap = g

    def tree_of(lengths):
        p = min_arborescence(n, r, lengths, tiebreak)
        return p, [(u, v) for v, u in enumerate(p) if u >= 0]

    w, _, rate, iters = _mwu(cap, tree_of, eps)
    return w, rate, iters


def mwu_allreduce(pairs, n, eps=0.1, tiebreak="asc"):
    """MWU packing of undirected spanning trees: Kruskal inner
    oracle, capacity per undirected link = per-direction capacity (R#9).
    Returns (weights {edge_tuple: w}, rate c*, iterations)."""
    def tree_of(lengths):
        t = min_spanning_tree(n, lengths, tiebreak)
        return t, list(t)

    w, _, rate, iters = _mwu(pairs, tree_of, eps)
    return w, rate, iters


# --------------------------------------------------------------------------
# Tree helpers
# --------------------------------------------------------------------------
def parent_depth(parent):
    """Max hops root -> leaf of a parent tuple."""
    best = 0
    for v in range(len(parent)):
        d, x = 0, v
        while parent[x] >= 0:
            x = parent[x]
            d += 1
        best = max(best, d)
    return best


def tree_centre(edges, n):
    """Centre of an undirected tree: minimum eccentricity, ties -> lowest id
    (R#9: "a chosen root vertex")."""
    adj = {v: [] for v in range(n)}
    for (u, v) in edges:
        adj[u].append(v)
        adj[v].append(u)

    def ecc(s):
        dist = {s: 0}
        frontier = [s]
        while frontier:
            nxt = []
            for u in frontier:
                for w in adj[u]:
                    if w not in dist:
                        dist[w] = dist[u] + 1
                        nxt.append(w)
            frontier = nxt
        return max(dist.values())

    return min(range(n), key=lambda v: (ecc(v), v))


def root_tree(edges, n, root):
    """Orient an undirected tree away from `root`: parent tuple."""
    adj = {v: [] for v in range(n)}
    for (u, v) in edges:
        adj[u].append(v)
        adj[v].append(u)
    parent = [None] * n
    parent[root] = -1
    stack = [root]
    while stack:
        u = stack.pop()
        for w in adj[u]:
            if parent[w] is None:
                parent[w] = u
                stack.append(w)
    return tuple(parent)


# --------------------------------------------------------------------------
# ILP refinement (Sec. 3.2.1)
# --------------------------------------------------------------------------
def ilp_refine(caps, candidates, c_star, gap=0.05, grids=(1, 2, 4, 8, 16), node_limit=500):
    """Eqs. 4-7 with the relaxation grid (R#5).

    `caps`: {edge: c_e}; `candidates`: list of (edge_list, depth, key) in a
    fixed order -- "k here is controlled by the number of trees returned by the
    MWU procedure".  For each g: maximise sum z_T s.t.
    sum_{T contains e} z_T <= g c_e, z_T in {0..g} (w_T = z_T / g <= 1, Eq. 6
    relaxed to the grid).  Tie-breaks (R#21): fewest trees, then the smallest
    maximum depth, then the least total depth (depth adds pipeline latency,
    P:511-513).  Accept the first g with sum z / g >= (1 - gap) c*.
    Returns (list of (candidate index, Fraction weight), g, accepted).
    scipy.optimize.milp (HiGHS) is the library primitive; the lexicographic
    tie-breaks are sequential MILPs."""
    from scipy.optimize import milp, LinearConstraint, Bounds

    edges = sorted(caps)
    eidx = {e: i for i, e in enumerate(edges)}
    k = len(candidates)
    A = np.zeros((len(edges), k))
    for j, (te, _, _) in enumerate(candidates):
        for e in te:
            A[eidx[e], j] += 1.0
    cvec = np.array([caps[e] for e in edges], dtype=float)
    depth = np.array([d for (_, d, _) in candidates], dtype=float)
    best = None
    for g in grids:
        # variables: z (k, integer 0..g), y (k, binary: tree used), D (max depth)
        Z = np.hstack([A, np.zeros_like(A), np.zeros((len(edges), 1))])
        link = np.hstack([np.eye(k), -g * np.eye(k), np.zeros((k, 1))])       # z_T <= g y_T
        dmax = np.hstack([np.zeros((k, k)), np.diag(depth), -np.ones((k, 1))])  # depth_T y_T <= D
        cons = [LinearConstraint(Z, -np.inf, g * cvec), LinearConstraint(link, -np.inf, 0.0),
                LinearConstraint(dmax, -np.inf, 0.0)]
        integ = np.concatenate([np.ones(2 * k), [0]])
        bnds = Bounds(np.zeros(2 * k + 1), np.concatenate([np.full(k, g), np.ones(k), [np.inf]]))
        ones_z = np.concatenate([np.ones(k), np.zeros(k), [0]])
        ones_y = np.concatenate([np.zeros(k), np.ones(k), [0]])
        d_max = np.concatenate([np.zeros(2 * k), [1]])
        dep_y = np.concatenate([np.zeros(k), depth, [0]])
        r1 = milp(-ones_z, constraints=cons, integrality=integ, bounds=bnds)
        zstar = round(-r1.fun)
        x = r1.x
        # tie-breaks as sequential MILPs under a deterministic node limit; a
        # limit-stopped stage keeps its best feasible point (the tie-break is
        # a preference, not a pin).
        cons.append(LinearConstraint(ones_z[None, :], zstar, zstar))
        for obj in (ones_y, d_max, dep_y):
            r = milp(obj, constraints=cons, integrality=integ, bounds=bnds,
                     options={"node_limit": node_limit})
            if r.x is None:
                break
            x = r.x
            val = float(obj @ np.round(x))
            cons.append(LinearConstraint(obj[None, :], -np.inf, val + 1e-6))
        z = np.round(x[:k]).astype(int)
        sol = [(j, Fraction(int(z[j]), g)) for j in range(k) if z[j] > 0]
        cur = (sol, g, zstar / g >= (1 - gap) * c_star - 1e-12)
        if cur[2]:
            return cur
        if best is None or sum(w for _, w in cur[0]) > sum(w for _, w in best[0]):
            best = cur              # not accepted anywhere: the best rate seen
    return best


# --------------------------------------------------------------------------
# MWU candidate sets: several MWU runs widen the candidates the ILP
# chooses from (SURVEY 7 hard part 8: "a larger candidate set from several
# eps/tie-break runs"); c* is the best MWU rate among them (R#3).
# --------------------------------------------------------------------------
MWU_RUNS = ((0.1, "asc"), (0.1, "desc"), (0.05, "asc"), (0.05, "desc"))


def optimal_rate(g, allreduce, r, c_star_mwu):
    """The rate the ILP's relaxation is measured against ("within a
    configured threshold ... of c*", c* = b* = "the optimal rate"; R#3).
    MWU only approximates it from below ((1 - eps)), so where the
    optimum is exactly computable it is used: Broadcast -- Edmonds' theorem,
    min_v maxflow(r -> v); AllReduce -- the Nash-Williams partition
    bound by enumeration for <= 8 GPUs (Bell(8) = 4140 partitions).  Larger
    AllReduce allocations fall back to the best MWU rate."""
    from . import bounds
    from .graphs import undirected_pairs
    n, _ = g
    if not allreduce:
        return float(bounds.edmonds_rate(g, r))
    if n <= 8:
        return float(bounds.nash_williams_rate(undirected_pairs(g), n))
    return c_star_mwu


def mwu_runs(eps):
    """The MWU runs of one plan: the configured eps with both tie-breaks, then
    eps / 2 with both (the defaults give MWU_RUNS)."""
    return ((eps, "asc"), (eps, "desc"), (eps / 2, "asc"), (eps / 2, "desc"))


def _order_trees(trees):
    """Split order (R#11): weight descending, then lexicographic edge list."""
    return sorted(trees, key=lambda t: (-t["weight"], sorted(t["edges"])))


def plan_broadcast_graph(g, r, eps=0.1, gap=0.05):
    """Broadcast plan on an explicit link graph: MWU then ILP (Secs. 3.2, 3.2.1).
    Candidates = the union of the trees of the MWU runs (`mwu_runs`); c* = the
    best MWU rate.  Returns dict(trees=[{parent, root, weight(Fraction), edges,
    depth}], rate, c_star, grid, accepted)."""
    n, cap = g
    if n == 1:
        return dict(trees=[dict(parent=(-1,), root=0, weight=Fraction(1), edges=[], depth=0)],
                    rate=Fraction(1), c_star=1.0)
    cands, c_star = set(), 0.0
    for e, tb in mwu_runs(eps):
        w, rate, _ = mwu_broadcast(g, r, e, tb)
        cands |= set(w)
        c_star = max(c_star, rate)
    cands = sorted(cands)                                  # parent tuples
    cand = [([(u, v) for v, u in enumerate(p) if u >= 0], parent_depth(p), p) for p in cands]
    opt = optimal_rate(g, False, r, c_star)
    sol, gg, ok = ilp_refine(cap, cand, opt, gap)
    trees = []
    for j, wt in sol:
        p = cands[j]
        trees.append(dict(parent=p, root=r, weight=wt, edges=cand[j][0], depth=cand[j][1]))
    trees = _order_trees(trees)
    return dict(trees=trees, rate=sum(t["weight"] for t in trees), c_star=c_star, opt=opt, grid=gg,
                accepted=ok)


def plan_allreduce_graph(g, eps=0.1, gap=0.05):
    """AllReduce plan on an explicit link graph: undirected MWU runs then ILP;
    each tree rooted at its centre (Sec. 3.3)."""
    from .graphs import undirected_pairs
    n, cap = g
    if n == 1:
        return dict(trees=[dict(parent=(-1,), root=0, weight=Fraction(1), edges=[], depth=0)],
                    rate=Fraction(1), c_star=1.0)
    pairs = undirected_pairs(g)
    cands, c_star = set(), 0.0
    for e, tb in mwu_runs(eps):
        w, rate, _ = mwu_allreduce(pairs, n, e, tb)
        cands |= set(w)
        c_star = max(c_star, rate)
    cands = sorted(cands)
    cand = []
    for t in cands:
        root = tree_centre(t, n)
        cand.append((list(t), parent_depth(root_tree(t, n, root)), t))
    opt = optimal_rate(g, True, 0, c_star)
    sol, gg, ok = ilp_refine(pairs, cand, opt, gap)
    trees = []
    for j, wt in sol:
        t = cands[j]
        root = tree_centre(t, n)
        trees.append(dict(parent=root_tree(t, n, root), root=root, weight=wt,
                          edges=list(t), depth=cand[j][1]))
    trees = _order_trees(trees)
    return dict(trees=trees, rate=sum(t["weight"] for t in trees), c_star=c_star, opt=opt, grid=gg,
                accepted=ok)


def plan_switch_allreduce(m):
    """Sec. 3.5: "with m GPUs, each GPU acts as a root for 1/m of
    the data chunks and each root is directly connected to (m - 1) leaf nodes,
    resulting in m one-hop trees".  Tree j = star centred at j, weight 1/2 in
    K_m link units (Nash-Williams optimum m/2, R#10).  Order: root rank."""
    trees = []
    for j in range(m):
        parent = tuple(-1 if v == j else j for v in range(m))
        trees.append(dict(parent=parent, root=j, weight=Fraction(1, 2),
                          edges=[(min(j, v), max(j, v)) for v in range(m) if v != j], depth=1 if m > 1 else 0))
    return dict(trees=trees, rate=Fraction(m, 2), c_star=m / 2)


def plan_switch_broadcast(m, r, onehop=False):
    """Switch Broadcast (R#10; the paper covers only AllReduce on a switch):
    the m - 1 two-level trees r -> k -> (all others), weight 1 each (Edmonds
    optimum m - 1 on K_m), ordered by k; or, for small buffers, the single
    one-hop star r -> all."""
    if m == 1:
        return dict(trees=[dict(parent=(-1,), root=0, weight=Fraction(1), edges=[], depth=0)], rate=Fraction(1))
    if onehop or m == 2:
        parent = tuple(-1 if v == r else r for v in range(m))
        return dict(trees=[dict(parent=parent, root=r, weight=Fraction(1),
                                edges=[(r, v) for v in range(m) if v != r], depth=1)], rate=Fraction(1))
    trees = []
    for k in range(m):
        if k == r:
            continue
        parent = tuple(-1 if v == r else (r if v == k else k) for v in range(m))
        trees.append(dict(parent=parent, root=r, weight=Fraction(1),
                          edges=[(p, v) for v, p in enumerate(parent) if p >= 0], depth=2))
    return dict(trees=trees, rate=Fraction(m - 1))


def plan_shallow(g, allreduce, r=0):
    """Latency plan for small calls on link graphs (R#27): ONE minimum-depth
    tree.  The paper: a chunk waits for the whole chunk at every hop, so depth
    adds latency, and on the switch it uses depth-1 trees
    (P:440-444).  Level sets L_0 = {root}, L_{k+1} = vertices not yet reached
    with a link from L_k (Broadcast: directed u -> v; AllReduce: both
    directions present); parent(v) = the lowest-rank u in the previous level
    with a link u -> v.  AllReduce roots the tree at the graph centre: the
    vertex whose level sets end soonest (minimum eccentricity), ties -> the
    lowest rank (R#9's rule)."""
    n, cap = g

    def link(u, v):
        return cap.get((u, v), 0) > 0 and (not allreduce or cap.get((v, u), 0) > 0)

    def levels(src):
        seen, lev, out = {src}, [src], [[src]]
        while True:
            nxt = sorted({v for u in lev for v in range(n) if v not in seen and link(u, v)})
            if not nxt:
                return out, seen
            seen |= set(nxt)
            out.append(nxt)
            lev = nxt

    if allreduce:
        best = None
        for s in range(n):
            lv, seen = levels(s)
            if len(seen) == n and (best is None or len(lv) < best[0]):
                best = (len(lv), s)
        if best is None:
            raise ValueError("graph not connected over bidirectional links")
        r = best[1]
    lv, seen = levels(r)
    if len(seen) != n:
        raise ValueError("rank unreachable from the root")
    parent = [-1] * n
    for k in range(1, len(lv)):
        for v in lv[k]:
            parent[v] = min(u for u in lv[k - 1] if link(u, v))
    edges = [(min(u, v), max(u, v)) if allreduce else (u, v) for v, u in enumerate(parent) if u >= 0]
    tree = dict(parent=tuple(parent), root=r, weight=Fraction(1), edges=edges, depth=len(lv) - 1)
    return dict(trees=[tree], rate=Fraction(1))


def split_bytes(S, weights):
    """Weight-proportional split (R#11): G = floor(S/16) grains,
    b_i = floor(G * sum_{j<i} w_j / sum w); tree i gets bytes
    [16 b_i, 16 b_{i+1}); the last tree also gets the S mod 16 tail.
    Returns a list of (lo, hi) byte ranges."""
    ws = [Fraction(w) for w in weights]
    W = sum(ws)
    G = S // GRAIN
    b = []
    acc = Fraction(0)
    for w in ws:
        b.append(math.floor(G * acc / W))
        acc += w
    b.append(G)
    out = [(GRAIN * b[i], GRAIN * b[i + 1]) for i in range(len(ws))]
    lo, _ = out[-1]
    out[-1] = (lo, S)
    return out


def link_load(plan, n, allreduce):
    """Per-GPU max(egress, ingress) in units of S for a plan:
    Broadcast edges carry S_i once; AllReduce edges carry S_i in each direction."""
    egress = [Fraction(0)] * n
    ingress = [Fraction(0)] * n
    W = sum(t["weight"] for t in plan["trees"])
    for t in plan["trees"]:
        f = t["weight"] / W
        for v, p in enumerate(t["parent"]):
            if p < 0:
                continue
            egress[p] += f
            ingress[v] += f
            if allreduce:
                egress[v] += f
                ingress[p] += f
    return max(max(egress), max(ingress))


# --------------------------------------------------------------------------
# NEXT-4: three-phase multi-server AllReduce (Sec. 3.5, Fig.
# hierarchy-allreduce P:402-407)
# --------------------------------------------------------------------------
def _ecc(parent_edges, n, s):
    adj = {v: [] for v in range(n)}
    for (u, v) in parent_edges:
        adj[u].append(v)
        adj[v].append(u)
    dist = {s: 0}
    fr = [s]
    while fr:
        nx = []
        for u in fr:
            for w in adj[u]:
                if w not in dist:
                    dist[w] = dist[u] + 1
                    nx.append(w)
        fr = nx
    return max(dist.values())


def plan_multiserver_allreduce(g, servers, eps=0.1, gap=0.05):
    """Three-phase AllReduce as one set of spanning trees.

    P:453: "we first partition data based on the number of spanning trees we
    have" -- K partitions, K = min over servers of the local packing's tree
    count (R#24: equal partitions, since one partition spans every server).
    Phase 1: per-server reduction over the local tree T_{s,p} to its
    server-local root r_{s,p}; "Each data partition has a distinct
    server-local root" -- R#25: roots chosen by minimum eccentricity
    among the server's GPUs not yet used as a root, ties -> lowest id.
    Phase 2: "across n servers, there are n one-hop cross-server
    trees, with each server-local root connected to (n - 1) roots on other
    servers" -- partition p splits into n sub-slices, sub-slice q rooted at
    r_{q,p}.  Phase 3: r_{s,p} broadcasts down T_{s,p}.
    Tree (p, q) = union of the T_{s,p} oriented to r_{s,p} plus r_{s,p} ->
    r_{q,p}; AllReduce on it performs all three phases per chunk.
    `servers`: list of lists of global GPU ids.  Returns a plan dict."""
    from .graphs import induced
    n_gpu = g[0]
    local = []
    for ids in servers:
        ids = sorted(ids)
        if len(ids) == 1:
            local.append((ids, None))
        else:
            sub, _ = induced(g, ids)
            local.append((ids, plan_allreduce_graph(sub, eps, gap)))
    counts = [len(p["trees"]) for _, p in local if p is not None]
    K = min(counts) if counts else 1
    # per server, per partition: (global edges, local root)
    parts = []
    for ids, lp in local:
        row = []
        used = set()
        for p in range(K):
            if lp is None:
                row.append(([], ids[0]))
                continue
            t = lp["trees"][p]
            k = len(ids)
            cands = sorted(range(k), key=lambda v: (_ecc(t["edges"], k, v), v))
            pick = next((v for v in cands if v not in used), cands[0])
            used.add(pick)
            row.append(([(ids[a], ids[b]) for (a, b) in t["edges"]], ids[pick]))
        parts.append(row)
    trees = []
    for p in range(K):
        roots = [parts[s][p][1] for s in range(len(servers))]
        for q in range(len(servers)):
            edges = []
            for s in range(len(servers)):
                edges += parts[s][p][0]
            edges += [(roots[s], roots[q]) for s in range(len(servers)) if s != q]
            parent = root_tree(edges, n_gpu, roots[q])
            trees.append(dict(parent=parent, root=roots[q], weight=Fraction(1),
                              edges=edges, depth=parent_depth(parent), partition=p, server=q))
    return dict(trees=trees, rate=None, partitions=K)
