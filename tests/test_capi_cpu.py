"""CPU-only checks of the C-ABI library: it loads without a GPU, exports every
symbol include/blink.h declares, and its host-only control plane
(blink_plan_json) satisfies the oracle's invariants (feasibility, rate within
the ILP gap of the Edmonds / Nash-Williams optimum, exact splits) -- no compute
calls, no GPU."""
import ctypes
import os
import re
from fractions import Fraction

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "blink.h")


@pytest.fixture(scope="module")
def B():
    from paper_1910_04940_b200 import build
    build.build()
    import paper_1910_04940_b200 as B
    return B


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"\b(blink_[a-z_]+)\s*\(", txt)))


def test_header_declares_the_survey_boundary():
    syms = declared_symbols()
    for s in ("blink_init", "blink_init_all", "blink_export_handle", "blink_connect",
              "blink_broadcast", "blink_allreduce", "blink_get_plan", "blink_destroy",
              "blink_result_string", "blink_last_error", "blink_plan_json"):
        assert s in syms


def test_library_exports_every_declared_symbol(B):
    lib = ctypes.CDLL(B.LIB_PATH)
    for s in declared_symbols():
        assert hasattr(lib, s), s


def test_result_strings_and_defaults(B):
    lib = B._lib
    assert lib.blink_result_string(0) == b"success"
    assert lib.blink_result_string(10) == b"timeout"
    c = B.config()
    assert c.mwu_eps == 0.1 and c.ilp_gap == 0.05 and c.threads == 256
    assert c.nvls == 0 and c.nvls_bytes == 64 << 20 and c.shallow_max_bytes == 256 << 10


def _oracle_plan(p):
    return dict(trees=[dict(parent=tuple(t["parent"]), root=t["root"],
                            weight=Fraction(*t["weight"])) for t in p["trees"]])


_ORACLE_PLANS = {}


def _oracle_plan_for(g, allreduce, root):
    """The oracle's paper-faithful plan (MWU runs -> ILP ladder),
    cached per graph for the module."""
    from oracle import packing
    n, cap = g
    key = (n, tuple(sorted(cap.items())), allreduce, root)
    if key not in _ORACLE_PLANS:
        _ORACLE_PLANS[key] = packing.plan_allreduce_graph(g) if allreduce else packing.plan_broadcast_graph(g, root)
    return _ORACLE_PLANS[key]


def _check_against_paper_pipeline(p, g, allreduce, root):
    """The C++ plan against the oracle's paper pipeline: where the
    paper's procedure reaches the 5% threshold, the C++ plan reaches it too,
    with no more trees and no deeper trees; where it does not (Eq. 6's
    w <= 1 cannot use parallel links twice, R#26), the C++ rate is at least
    the oracle's."""
    o = _oracle_plan_for(g, allreduce, root)
    unit = min(g[1].values())
    crate = Fraction(*p["rate"]) * unit
    if o["accepted"]:
        assert p["accepted"]
        assert len(p["trees"]) <= len(o["trees"])
        assert max(t["depth"] for t in p["trees"]) <= max(t["depth"] for t in o["trees"])
    else:
        assert crate >= o["rate"]
    assert abs(p["opt"] * unit - o["opt"]) < 1e-9


def _check_plan(p, g, allreduce):
    """Plan weights are in units of the graph's smallest link capacity (R#23):
    scale by it before comparing with the raw-capacity optimum."""
    from oracle import bounds, graphs
    n, cap = g
    unit = min(cap.values())
    W = sum(Fraction(*t["weight"]) for t in p["trees"])
    assert Fraction(*p["rate"]) == W
    W = W * unit
    if allreduce:
        pairs = graphs.undirected_pairs(g)
        load = {e: Fraction(0) for e in pairs}
        for t in p["trees"]:
            for v, u in enumerate(t["parent"]):
                if u >= 0:
                    load[(min(u, v), max(u, v))] += Fraction(*t["weight"]) * unit
        assert all(load[e] <= pairs[e] for e in pairs)
        opt = bounds.nash_williams_rate(pairs, n)
    else:
        load = {e: Fraction(0) for e in cap}
        for t in p["trees"]:
            assert t["parent"][p["root"]] == -1
            for v, u in enumerate(t["parent"]):
                if u >= 0:
                    load[(u, v)] += Fraction(*t["weight"]) * unit
        assert all(load[e] <= cap[e] for e in cap)
        opt = bounds.edmonds_rate(g, p["root"])
    # rate within the ILP gap (5%) of the true optimum (R#3)
    assert float(W) >= 0.95 * opt - 1e-9
    # split: contiguous, 16-byte grains, covers [0, count)
    es = p["esize"]
    rngs = [(t["lo"], t["hi"]) for t in p["trees"]]
    assert rngs[0][0] == 0 and rngs[-1][1] == p["count"]
    for (a, b), (c, d) in zip(rngs, rngs[1:]):
        assert b == c and (a * es) % 16 == 0
    for t in p["trees"]:
        if t["hi"] > t["lo"]:
            assert t["nchunks"] == -(-(t["hi"] - t["lo"]) // t["chunk"])


@pytest.mark.parametrize("root", range(8))
def test_dgx1v_broadcast_plan_is_six_unit_trees(B, root):
    from oracle import graphs
    g = graphs.dgx1v()
    p = B.plan_json(8, False, root, 1000 * 10**6 // 4, "f32", graph=B.Graph.from_pairs(8, g[1]))
    assert len(p["trees"]) == 6 and p["rate"] == [6, 1]
    assert all(t["weight"] == [1, 1] for t in p["trees"])
    _check_plan(p, g, False)
    _check_against_paper_pipeline(p, g, False, root)


@pytest.mark.parametrize("root", range(8))
def test_dgx1p_broadcast_plans(B, root):
    from oracle import graphs
    g = graphs.dgx1p()
    p = B.plan_json(8, False, root, 1 << 20, "f32", graph=B.Graph.from_pairs(8, g[1]))
    assert len(p["trees"]) == 4 and p["rate"] == [4, 1]           # Edmonds rate 4 (App. A)
    _check_plan(p, g, False)
    _check_against_paper_pipeline(p, g, False, root)


@pytest.mark.parametrize("name", ["dgx1v", "dgx1p"])
def test_dgx1_allreduce_plans(B, name):
    from oracle import graphs
    g = graphs.dgx1v() if name == "dgx1v" else graphs.dgx1p()
    p = B.plan_json(8, True, 0, (1 << 20) + 3, "f32", graph=B.Graph.from_pairs(8, g[1]))
    _check_plan(p, g, True)
    _check_against_paper_pipeline(p, g, True, 0)


FRAGMENTS = [[0, 1, 4], [0, 1, 3, 4, 5, 7], [2, 3, 6, 7], [1, 4, 5, 6]]


@pytest.mark.parametrize("machine", ["dgx1v", "dgx1p"])
@pytest.mark.parametrize("ids", FRAGMENTS)
def test_fragment_plans_match_or_beat_the_paper_pipeline(B, machine, ids):
    from oracle import graphs
    full = graphs.dgx1v() if machine == "dgx1v" else graphs.dgx1p()
    g, _ = graphs.induced(full, ids)
    n = g[0]
    packed = B.config(shallow_max_bytes=0)
    G = B.Graph.from_pairs(n, g[1])
    for allreduce in (False, True):
        p = B.plan_json(n, allreduce, 0, 123457, "f32", graph=G, cfg=packed)
        _check_plan(p, g, allreduce)
        _check_against_paper_pipeline(p, g, allreduce, 0)


def test_three_gpu_plans_match_the_oracle_exactly(B):
    from oracle import graphs, packing
    tri, _ = graphs.induced(graphs.dgx1p(), [0, 1, 3])
    G = B.Graph.from_pairs(3, tri[1])
    pb = B.plan_json(3, False, 0, 262144, "f32", graph=G)
    ob = packing.plan_broadcast_graph(tri, 0)
    assert {tuple(t["parent"]) for t in pb["trees"]} == {t["parent"] for t in ob["trees"]}
    pa = B.plan_json(3, True, 0, 262144, "f32", graph=G)
    oa = packing.plan_allreduce_graph(tri)
    assert [tuple(t["parent"]) for t in pa["trees"]] == [t["parent"] for t in oa["trees"]]
    assert [t["hi"] - t["lo"] for t in pa["trees"]] == [87380, 87380, 87384]


@pytest.mark.parametrize("m", [1, 2, 3, 5, 8, 16])
def test_switch_plans_equal_oracle_closed_forms(B, m):
    from oracle import collectives, packing
    count = 1000 * m + 7
    pa = B.plan_json(m, True, 0, count, "bf16")
    oa = packing.plan_switch_allreduce(m)
    assert [tuple(t["parent"]) for t in pa["trees"]] == [t["parent"] for t in oa["trees"]]
    assert [(t["lo"], t["hi"]) for t in pa["trees"]] == collectives.tree_element_ranges(oa, count, "bf16")
    if m > 2:
        pb = B.plan_json(m, False, m - 1, count, "f32")
        ob = packing.plan_switch_broadcast(m, m - 1)
        assert [tuple(t["parent"]) for t in pb["trees"]] == [t["parent"] for t in ob["trees"]]


@pytest.mark.parametrize("count", [0, 1, 3, 4, 5, 262144, 10**9 // 4 + 1])
def test_split_matches_oracle_for_weighted_trees(B, count):
    from oracle import collectives, graphs
    g = graphs.dgx1v()
    p = B.plan_json(8, True, 0, count, "f32", graph=B.Graph.from_pairs(8, g[1]))
    got = [(t["lo"], t["hi"]) for t in p["trees"]]
    assert got == collectives.tree_element_ranges(_oracle_plan(p), count, "f32")


def test_topology_errors(B):
    # dangling endpoint, nonpositive capacity, disconnected, missing reverse
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(3, False, 0, 16, graph=B.Graph(3, [(0, 1, 1, 1), (1, 9, 1, 1)]))
    assert e.value.code == 8 and "dangling" in str(e.value)
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(2, False, 0, 16, graph=B.Graph(2, [(0, 1, 0.0, 1)]))
    assert e.value.code == 8 and "capacity" in str(e.value)
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(4, False, 0, 16, graph=B.Graph(4, [(0, 1, 1, 1), (2, 3, 1, 1)]))
    assert e.value.code == 8 and "{2,3}" in str(e.value)
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(3, True, 0, 16, graph=B.Graph(3, [(0, 1, 1, 1), (1, 2, 1, 0), (2, 0, 1, 1)]))
    assert e.value.code == 8 and "reverse" in str(e.value)
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(3, False, 5, 16)
    assert e.value.code == 4


def test_switch_graph_with_switch_node(B):
    # 4 GPUs on one SWITCH node (node 4): one-hop trees
    G = B.Graph(4, [(v, 4, 6.0, 1) for v in range(4)], switches=1)
    p = B.plan_json(4, True, 0, 4096, "f32", graph=G)
    assert p["switch"] and len(p["trees"]) == 4 and p["rate"] == [2, 1]


@pytest.mark.parametrize("servers", [[[0, 1, 3], [2, 4, 5, 6, 7]], [[0, 1, 2, 3], [4, 5, 6, 7]],
                                     [[0, 1], [2, 3], [4, 5, 6, 7]]])
def test_multiserver_plans_follow_the_three_phase_protocol(B, servers):
    """NEXT-4: K partitions x n one-hop cross-server trees; same
    partition count and structure as the oracle's plan."""
    from oracle import graphs, packing
    g = graphs.dgx1v()
    where = {v: i for i, s in enumerate(servers) for v in s}
    cap = {(u, v): c for (u, v), c in g[1].items() if where[u] == where[v]}
    p = B.plan_json(8, True, 0, (1 << 20) + 5, "f32", graph=B.Graph.multi_server(8, g[1], servers))
    o = packing.plan_multiserver_allreduce((8, cap), servers)
    # K = the fewest trees of a server-local AllReduce plan (R#24), from the
    # library's own local plans (its product heuristics may pack a server
    # differently from the oracle's paper pipeline, R#21/R#26)
    packed = B.config(shallow_max_bytes=0)
    K = min(len(B.plan_json(len(ids), True, 0, 4096, "f32", cfg=packed,
                            graph=B.Graph.from_pairs(len(ids), graphs.induced(g, ids)[0][1]))["trees"])
            for ids in servers if len(ids) > 1)
    assert len(p["trees"]) == K * len(servers)
    assert len(o["trees"]) == o["partitions"] * len(servers)
    for i, t in enumerate(p["trees"]):
        q = i % len(servers)
        assert where[t["root"]] == q and t["parent"].count(-1) == 1
        cross = [(u, v) for v, u in enumerate(t["parent"]) if u >= 0 and where[u] != where[v]]
        assert len(cross) == len(servers) - 1
        assert all(u == t["root"] for u, v in cross)          # star into the sub-slice root
    rngs = [(t["lo"], t["hi"]) for t in p["trees"]]
    assert rngs[0][0] == 0 and rngs[-1][1] == (1 << 20) + 5


def test_multiserver_errors(B):
    # a server with no network attachment is disconnected; Broadcast unsupported
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(4, True, 0, 64, graph=B.Graph(4, [(0, 1, 1, 1), (2, 3, 1, 1), (0, 4, 1, 1)], switches=1))
    assert e.value.code == 8 and "{2,3}" in str(e.value)
    G = B.Graph(4, [(0, 1, 1, 1), (2, 3, 1, 1), (0, 4, 1, 1), (2, 4, 1, 1)], switches=1)
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(4, False, 0, 64, graph=G)
    assert e.value.code == 9
    assert len(B.plan_json(4, True, 0, 64, graph=G)["trees"]) == 2


@pytest.mark.parametrize("seed", range(24))
def test_random_graph_plans_satisfy_the_oracle_invariants(B, seed):
    """C++ control plane on random connected link graphs (2-7 GPUs, capacities
    1-3): Broadcast plans are arborescences from the root, AllReduce plans are
    spanning trees; both are feasible (Eqs. 2, 5), reach >= 95% of the
    Edmonds / Nash-Williams optimum and never exceed it, and match or beat the
    oracle's paper pipeline (trees, depth)."""
    import random
    from oracle import bounds, graphs
    rng = random.Random(4000 + seed)
    n = rng.randint(2, 7)
    while True:
        cap = {}
        for u in range(n):
            for v in range(u + 1, n):
                if rng.random() < 0.55:
                    c = rng.randint(1, 3)
                    cap[(u, v)] = cap[(v, u)] = c
        if graphs.is_connected((n, cap)):
            break
    G = B.Graph.from_pairs(n, cap)
    root = rng.randrange(n)
    packed = B.config(shallow_max_bytes=0)  # the packed plan at every size (not R#27's small-call tree)
    pb = B.plan_json(n, False, root, 123457, "f32", graph=G, cfg=packed)
    _check_plan(pb, (n, cap), False)
    for t in pb["trees"]:
        par = t["parent"]
        assert par[root] == -1 and all((par[v], v) in cap for v in range(n) if v != root)
    unit = min(cap.values())
    assert Fraction(*pb["rate"]) * unit <= bounds.edmonds_rate((n, cap), root) + Fraction(1, 10**9)
    _check_against_paper_pipeline(pb, (n, cap), False, root)
    pa = B.plan_json(n, True, 0, 123457, "bf16", graph=G, cfg=packed)
    _check_plan(pa, (n, cap), True)
    _check_against_paper_pipeline(pa, (n, cap), True, 0)
    pairs = graphs.undirected_pairs((n, cap))
    assert float(Fraction(*pa["rate"]) * unit) <= bounds.nash_williams_rate(pairs, n) + 1e-9
    for t in pa["trees"]:
        par = t["parent"]
        assert par.count(-1) == 1
        assert all((min(par[v], v), max(par[v], v)) in pairs for v in range(n) if par[v] >= 0)


def test_init_all_rejects_too_many_ranks_before_touching_cuda(B):
    import ctypes
    hs = (ctypes.c_void_p * 17)()
    devs = (ctypes.c_int * 17)(*([0] * 17))
    assert B._lib.blink_init_all(hs, 17, devs, None, None) == 9       # BLINK_ERR_UNSUPPORTED
    assert b"16" in B._lib.blink_last_error(None)


@pytest.mark.parametrize("name", ["switch8", "dgx1v", "dgx1p", "tri"])
def test_library_plans_move_the_bytes_of_the_message_bound(B, name):
    """The library's plans, evaluated with the oracle's byte model
    (oracle/model.py, pinned in test_oracle_model.py): Broadcast moves
    (m-1) S and every non-root receives exactly S; AllReduce moves 2 (m-1) S
    (P:397-400)."""
    from oracle import graphs, model
    if name == "switch8":
        m, G = 8, None
    elif name == "tri":
        sub, _ = graphs.induced(graphs.dgx1p(), [0, 1, 3])
        m, G = 3, B.Graph.from_pairs(3, sub[1])
    else:
        g = graphs.dgx1v() if name == "dgx1v" else graphs.dgx1p()
        m, G = 8, B.Graph.from_pairs(8, g[1])
    count = 250001
    S = count * 4
    pb = _oracle_plan(B.plan_json(m, False, m - 1, count, "f32", graph=G))
    lb = model.link_bytes(pb, m, S, False)
    assert sum(lb.values()) == (m - 1) * S
    for v in range(m):
        assert sum(b for (_, w), b in lb.items() if w == v) == (0 if v == m - 1 else S)
    pa = _oracle_plan(B.plan_json(m, True, 0, count, "f32", graph=G))
    assert sum(model.link_bytes(pa, m, S, True).values()) == 2 * (m - 1) * S


# ------------------------------------------------------------ R#27 latency plan
def _bfs_dist_fw(n, cap, allreduce):
    """All-pairs hop distances by Floyd-Warshall (independent of the BFS)."""
    INF = 10**9
    d = [[0 if u == v else INF for v in range(n)] for u in range(n)]
    for (u, v), c in cap.items():
        if c > 0 and (not allreduce or cap.get((v, u), 0) > 0):
            d[u][v] = 1
    for k in range(n):
        for i in range(n):
            for j in range(n):
                if d[i][k] + d[k][j] < d[i][j]:
                    d[i][j] = d[i][k] + d[k][j]
    return d


@pytest.mark.parametrize("seed", range(12))
def test_small_calls_take_the_oracle_shallow_tree(B, seed):
    """Calls <= shallow_max_bytes on link graphs run on one minimum-depth tree
    (R#27): the C++ plan equals the oracle's plan_shallow, and every vertex
    sits at its shortest-path distance (Floyd-Warshall) from the root; the
    AllReduce root has the minimum eccentricity.  Above the threshold the
    packed plan returns."""
    import random
    from oracle import graphs, packing
    rng = random.Random(7000 + seed)
    n = rng.randint(3, 8)
    while True:
        cap = {}
        for u in range(n):
            for v in range(u + 1, n):
                if rng.random() < 0.45:
                    cap[(u, v)] = cap[(v, u)] = rng.randint(1, 3)
        if graphs.is_connected((n, cap)):
            break
    G = B.Graph.from_pairs(n, cap)
    root = rng.randrange(n)
    for allreduce in (False, True):
        p = B.plan_json(n, allreduce, root, 1000, "f32", graph=G)
        want = packing.plan_shallow((n, cap), allreduce, root)["trees"][0]
        assert len(p["trees"]) == 1
        t = p["trees"][0]
        assert tuple(t["parent"]) == want["parent"] and t["root"] == want["root"]
        d = _bfs_dist_fw(n, cap, allreduce)
        r = t["root"]
        if allreduce:
            assert max(d[r]) == min(max(row) for row in d)
        else:
            assert r == root
        assert t["depth"] == max(d[r][v] for v in range(n))
        for v in range(n):  # parent one level up, over a real link
            u = t["parent"][v]
            if v == r:
                assert u == -1
            else:
                assert d[r][u] + 1 == d[r][v] and cap.get((u, v), 0) > 0
        assert t["lo"] == 0 and t["hi"] == 1000
        # above the threshold: the packed plan (the size-independent count-0 plan)
        big = B.plan_json(n, allreduce, root, (256 << 10) // 4 + 1, "f32", graph=G)
        packed = B.plan_json(n, allreduce, root, 0, "f32", graph=G)
        assert [x["parent"] for x in big["trees"]] == [x["parent"] for x in packed["trees"]]


def test_dgx1v_small_broadcast_tree_golden(B):
    """App. B DGX-1V, root 0: neighbours 1, 2, 3, 4 at depth 1; 5, 6, 7 hang
    off their lowest-rank neighbour at depth 1 (1, 2, 3) -- derived by hand
    from the link list (P:56-61 reconstruction)."""
    from oracle import graphs, packing
    g = graphs.dgx1v()
    want = (-1, 0, 0, 0, 0, 1, 2, 3)
    assert packing.plan_shallow(g, False, 0)["trees"][0]["parent"] == want
    assert packing.plan_shallow(g, True)["trees"][0]["parent"] == want  # centre: rank 0 (all ecc 2)
    assert packing.plan_shallow(g, False, 5)["trees"][0]["parent"] == (1, 5, 1, 1, 5, -1, 5, 5)
    G = B.Graph.from_pairs(8, g[1])
    assert tuple(B.plan_json(8, False, 0, 4096, "f32", graph=G)["trees"][0]["parent"]) == want
    assert len(B.plan_json(8, False, 0, 1 << 20, "f32", graph=G)["trees"]) == 6
    assert len(B.plan_json(8, False, 0, 0, "f32", graph=G)["trees"]) == 6  # count 0: packed plan
    off = B.config(shallow_max_bytes=0)
    assert len(B.plan_json(8, False, 0, 4096, "f32", graph=G, cfg=off)["trees"]) == 6


def test_chunk_policy_deep_trees_and_merged_medium_calls(B):
    """a8 static table as documented in DESIGN §1: multi-hop Broadcast trees
    get a chunk floor of bytes/16 clamped to [16 KiB, 96 KiB] on link graphs
    and [16 KiB, 64 KiB] on the switch's two-level trees; chunk sizes are
    16-byte grains and the chunks cover every tree's range."""
    from oracle import graphs
    g = graphs.dgx1v()
    G = B.Graph.from_pairs(8, g[1])
    count = (64 << 20) // 4
    p = B.plan_json(8, False, 0, count, "f32", graph=G)
    for t in p["trees"]:
        nbytes = (t["hi"] - t["lo"]) * 4
        assert t["depth"] >= 2
        assert t["chunk"] * 4 >= min(96 << 10, max(16 << 10, nbytes // 16))
        assert (t["chunk"] * 4) % 16 == 0 and t["nchunks"] * t["chunk"] >= t["hi"] - t["lo"]
        assert t["chunk"] * 4 == 96 << 10   # ~11 MB trees: the cap binds (the per-CTA target is smaller)
    p = B.plan_json(8, False, 0, count, "f32")  # switch: 7 two-level trees
    assert len(p["trees"]) == 7
    for t in p["trees"]:
        nbytes = (t["hi"] - t["lo"]) * 4
        assert min(64 << 10, max(16 << 10, nbytes // 16)) <= t["chunk"] * 4
        assert t["chunk"] * 4 == 64 << 10
    # small trees: the floor follows the range (bytes / 16), never below 16 KiB
    p = B.plan_json(8, False, 0, (1 << 20) // 4, "f32", graph=G)
    for t in p["trees"]:
        nbytes = (t["hi"] - t["lo"]) * 4
        assert t["chunk"] * 4 >= max(16 << 10, nbytes // 16)


# ------------------------------------------------------------ NEXT-3 on link graphs
def _random_link_graph(seed, lo=3, hi=8, p=0.45):
    import random
    from oracle import graphs
    rng = random.Random(seed)
    n = rng.randint(lo, hi)
    while True:
        cap = {}
        for u in range(n):
            for v in range(u + 1, n):
                if rng.random() < p:
                    cap[(u, v)] = cap[(v, u)] = rng.randint(1, 3)
        if graphs.is_connected((n, cap)):
            return n, cap, rng


@pytest.mark.parametrize("seed", list(range(10)) + ["dgx1v", "dgx1p"])
def test_link_graph_allgather_and_gather_plans(B, seed):
    """NEXT-3 on packed link graphs.  AllGather: tree j is a spanning
    arborescence rooted at j over real links with every rank at its shortest
    distance from j (Floyd-Warshall) and covers block j.  Gather to r: tree j
    is a chain from j to r over real links of length dist(j, r), ranks off
    the chain are not members; tree r is r alone."""
    from oracle import graphs
    if seed in ("dgx1v", "dgx1p"):
        g = graphs.dgx1v() if seed == "dgx1v" else graphs.dgx1p()
        n, cap = g
        roots = range(n)
    else:
        n, cap, rng = _random_link_graph(9000 + seed)
        roots = [rng.randrange(n)]
    G = B.Graph.from_pairs(n, cap)
    d = _bfs_dist_fw(n, cap, False)
    count = 1001
    ag = B.plan_json(n, 3, 0, count, "f32", graph=G)
    assert len(ag["trees"]) == n
    for j, t in enumerate(ag["trees"]):
        par = t["parent"]
        assert t["root"] == j and par[j] == -1
        assert (t["lo"], t["hi"]) == (j * count, (j + 1) * count)
        for v in range(n):
            if v != j:
                assert cap.get((par[v], v), 0) > 0 and d[j][par[v]] + 1 == d[j][v]
        assert t["depth"] == max(d[j])
    for r in roots:
        ga = B.plan_json(n, 4, r, count, "f32", graph=G)
        assert len(ga["trees"]) == n
        for j, t in enumerate(ga["trees"]):
            par = t["parent"]
            assert t["root"] == j and par[j] == -1
            assert (t["lo"], t["hi"]) == (j * count, (j + 1) * count)
            members = [v for v in range(n) if par[v] != -2]
            assert len(members) == d[j][r] + 1 and t["depth"] == d[j][r]
            v = r
            while v != j:                      # walk back from the gather root
                u = par[v]
                assert cap.get((u, v), 0) > 0 and d[u][r] == d[v][r] + 1
                v = u


@pytest.mark.parametrize("seed", list(range(6)) + ["dgx1v"])
def test_link_graph_reduce_scatter_plans(B, seed):
    """ReduceScatter on link graphs (NEXT-3): tree j is a spanning tree rooted
    at j over bidirectional links, every rank at its shortest (undirected)
    distance from j, covering block j; a link without its reverse is a
    topology error."""
    from oracle import graphs
    if seed == "dgx1v":
        n, cap = graphs.dgx1v()
    else:
        n, cap, _ = _random_link_graph(9100 + seed)
    G = B.Graph.from_pairs(n, cap)
    d = _bfs_dist_fw(n, cap, True)
    p = B.plan_json(n, 2, 0, 777, "bf16", graph=G)
    assert len(p["trees"]) == n
    for j, t in enumerate(p["trees"]):
        par = t["parent"]
        assert t["root"] == j and par[j] == -1 and (t["lo"], t["hi"]) == (j * 777, (j + 1) * 777)
        for v in range(n):
            if v != j:
                u = par[v]
                assert cap.get((u, v), 0) > 0 and cap.get((v, u), 0) > 0 and d[j][u] + 1 == d[j][v]
    with pytest.raises(B.BlinkError) as e:
        B.plan_json(3, 2, 0, 16, graph=B.Graph(3, [(0, 1, 1, 1), (1, 2, 1, 0), (2, 0, 1, 1)]))
    assert e.value.code == 8 and "reverse" in str(e.value)


# ------------------------------------------------------------ topology probe
def _bus(i):
    return f"0000:{0x10 + 0x10 * i:02X}:00.0"


def _fake_table(path, ports):
    with open(path, "w") as f:
        for gpu, port, remote in ports:
            f.write(f"{gpu} {port} {remote}\n")


def test_probe_builds_the_dgx1v_graph_from_a_port_table(B, tmp_path, monkeypatch):
    """An injected NVML port table with DGX-1V's cabling (App. B: every GPU 6
    ports, 8 pairs doubled) must probe as kind "nvlink" with exactly the
    DGX-1V link multiplicities; NVML's bus-id spelling (8-digit domain) must
    match CUDA's."""
    from oracle import graphs
    n, cap = graphs.dgx1v()
    ports = []
    nxt = [0] * n
    for (u, v), c in sorted(cap.items()):
        for _ in range(c):
            ports.append((_bus(u).replace("0000:", "00000000:"), nxt[u], _bus(v)))
            nxt[u] += 1
    assert all(k == 6 for k in nxt)
    _fake_table(tmp_path / "t.txt", ports)
    monkeypatch.setenv("BLINK_FAKE_NVML", str(tmp_path / "t.txt"))
    d = B.topology_json([_bus(i) for i in range(n)])
    assert d["kind"] == "nvlink" and d["switch_ports"] == [0] * n
    got = {(u, v): c for u, v, c in d["links"]}
    assert got == dict(cap)


def test_probe_nvswitch_virtual_and_outside_gpus(B, tmp_path, monkeypatch):
    # 4 B200-like GPUs, 18 ports each, all ending at NVSwitches
    ports = [(_bus(i), p, "switch") for i in range(4) for p in range(18)]
    _fake_table(tmp_path / "s.txt", ports)
    monkeypatch.setenv("BLINK_FAKE_NVML", str(tmp_path / "s.txt"))
    d = B.topology_json([_bus(i) for i in range(4)])
    assert d["kind"] == "nvswitch" and d["switch_ports"] == [18] * 4 and d["links"] == []
    # one device repeated (virtual ranks): no NVML needed
    assert B.topology_json([_bus(0)] * 3)["kind"] == "virtual"
    # links to a GPU outside the allocation do not count; a pair
    # with ports only in one direction table still counts per direction
    ports = [(_bus(0), 0, _bus(1)), (_bus(1), 0, _bus(0)), (_bus(1), 1, _bus(2)), (_bus(2), 0, _bus(1)),
             (_bus(2), 1, _bus(7))]
    _fake_table(tmp_path / "c.txt", ports)
    monkeypatch.setenv("BLINK_FAKE_NVML", str(tmp_path / "c.txt"))
    d = B.topology_json([_bus(i) for i in range(3)])
    assert d["kind"] == "nvlink"
    assert sorted(tuple(x) for x in d["links"]) == [(0, 1, 1), (1, 0, 1), (1, 2, 1), (2, 1, 1)]
    with pytest.raises(B.BlinkError) as e:
        B.topology_json(["not-a-bus-id", _bus(1)])
    assert e.value.code == 4


def test_hybrid_split_matches_the_oracle(B):
    """blink_hybrid_split (Eq. 8) against oracle.model.hybrid_split, within the
    16-byte rounding of R#11; errors for bad arguments."""
    from fractions import Fraction
    from oracle import model
    for D, bp, bn, t in ((10**9, 32e9, 150e9, 1e-3), (3 * 10**8, 16e9, 50e9, 5e-4), (12345678, 25e9, 300e9, 0.0),
                         (10**6, 32e9, 150e9, 1.0)):
        dp, dn = B.hybrid_split(D, bp, bn, t)
        wp, wn = model.hybrid_split(D, Fraction(bp), Fraction(bn), Fraction(t))
        assert dp + dn == D and dp % 16 == 0
        assert wp - 16 <= dp <= wp + 1e-6 * D / 1e6 + 1
    with pytest.raises(B.BlinkError) as e:
        B.hybrid_split(100, 0.0, 1.0, 0.0)
    assert e.value.code == 4
