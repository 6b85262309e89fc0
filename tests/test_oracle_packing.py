"""Pins for oracle/bounds.py and oracle/packing.py.

Independent anchors: the paper's worked examples (tests/golden/paper_pins.json),
the Edmonds and Nash-Williams theorems checked against a brute-force LP over
every enumerated tree, brute-force minimum arborescences on tiny graphs, and
closed forms (K_m, one-hop split)."""
import json
import os
import random
from fractions import Fraction
from itertools import product

import numpy as np
import pytest

import synth

from oracle import bounds, graphs, packing

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def random_digraph(rng, n, p=0.6, cmax=3):
    while True:
        cap = {}
        for u in range(n):
            for v in range(n):
                if u != v and rng.random() < p:
                    cap[(u, v)] = rng.randint(1, cmax)
        g = (n, cap)
        if all(bounds.maxflow(n, cap, 0, v) > 0 for v in range(1, n)):
            return g


def random_undirected(rng, n, p=0.6, cmax=3):
    while True:
        pairs = {}
        for u in range(n):
            for v in range(u + 1, n):
                if rng.random() < p:
                    pairs[(u, v)] = rng.randint(1, cmax)
        cap = {}
        for (u, v), c in pairs.items():
            cap[(u, v)] = c
            cap[(v, u)] = c
        if graphs.is_connected((n, cap)):
            return pairs


# ----------------------------------------------------------------- bounds
@pytest.mark.parametrize("seed", range(12))
def test_edmonds_equals_brute_lp(seed):
    rng = random.Random(seed)
    g = random_digraph(rng, rng.randint(2, 5))
    r = rng.randrange(g[0])
    if not all(bounds.maxflow(g[0], g[1], r, v) > 0 for v in range(g[0]) if v != r):
        r = 0
    assert abs(bounds.edmonds_rate(g, r) - bounds.brute_broadcast_rate(g, r)) < 1e-7


@pytest.mark.parametrize("seed", range(12))
def test_nash_williams_equals_brute_lp(seed):
    rng = random.Random(100 + seed)
    n = rng.randint(2, 6)
    pairs = random_undirected(rng, n)
    assert abs(bounds.nash_williams_rate(pairs, n) - bounds.brute_allreduce_rate(pairs, n)) < 1e-7


def test_closed_forms_Km():
    for m in (2, 3, 4, 5):
        g = graphs.complete(m)
        assert bounds.edmonds_rate(g, 0) == m - 1
        pairs = graphs.undirected_pairs(g)
        assert abs(bounds.nash_williams_rate(pairs, m) - m / 2) < 1e-12
        assert abs(bounds.brute_allreduce_rate(pairs, m) - m / 2) < 1e-7
    assert abs(bounds.nash_williams_rate(graphs.undirected_pairs(graphs.complete(8)), 8) - 4) < 1e-12


def test_dgx1_rates():
    # DGX-1V broadcast rate 6 from every root (6 trees of rate 1.0)
    for r in range(8):
        assert bounds.edmonds_rate(graphs.dgx1v(), r) == 6
        assert bounds.edmonds_rate(graphs.dgx1p(), r) == 4
    # AllReduce (undirected): NW 24/7 (V), 16/7 (P) = 4 rings x 8/14 = 32/14
    assert abs(bounds.nash_williams_rate(graphs.undirected_pairs(graphs.dgx1p()), 8) - 32 / 14) < 1e-12
    assert abs(bounds.nash_williams_rate(graphs.undirected_pairs(graphs.dgx1v()), 8) - 24 / 7) < 1e-12


@pytest.mark.slow
def test_dgx1v_brute_lp_is_6():
    assert abs(bounds.brute_broadcast_rate(graphs.dgx1v(), 0) - 6) < 1e-7


# ------------------------------------------------------------ min arborescence
def _brute_min_arb(g, r, lengths):
    best = None
    for parent in bounds.enumerate_arborescences(g, r):
        cost = sum(lengths[(p, v)] for v, p in enumerate(parent) if p >= 0)
        if best is None or cost < best[0] - 1e-12:
            best = (cost, parent)
    return best[0]


@pytest.mark.parametrize("tiebreak", ["asc", "desc"])
@pytest.mark.parametrize("seed", range(20))
def test_min_arborescence_matches_brute_force(seed, tiebreak):
    rng = random.Random(500 + seed)
    g = random_digraph(rng, rng.randint(2, 6), p=0.7)
    lengths = {e: rng.choice([0.0, 0.5, 1.0, 2.0, rng.random()]) for e in g[1]}
    parent = packing.min_arborescence(g[0], 0, lengths, tiebreak)
    cost = sum(lengths[(p, v)] for v, p in enumerate(parent) if p >= 0)
    assert abs(cost - _brute_min_arb(g, 0, lengths)) < 1e-12
    assert parent in set(bounds.enumerate_arborescences(g, 0))


def test_tiebreaks_pick_the_extreme_in_edges():
    """Equal lengths everywhere: with no cycle to contract, every vertex keeps
    its cheapest in-edge, the lexicographically smallest (asc) or largest
    (desc) one (the alternate run of SURVEY 7 hard part 8)."""
    # DAG 0 -> {1, 2, 3}, 1 -> {2, 3}, 2 -> 3: all lengths 1
    L = {(0, 1): 1, (0, 2): 1, (0, 3): 1, (1, 2): 1, (1, 3): 1, (2, 3): 1}
    assert packing.min_arborescence(4, 0, L, "asc") == (-1, 0, 0, 0)
    assert packing.min_arborescence(4, 0, L, "desc") == (-1, 0, 1, 2)
    pairs = {(0, 1): 1.0, (0, 2): 1.0, (1, 2): 1.0}
    assert packing.min_spanning_tree(3, pairs, "asc") == ((0, 1), (0, 2))
    assert packing.min_spanning_tree(3, pairs, "desc") == ((0, 2), (1, 2))


def test_min_arborescence_spec_examples():
    # 3-cycle a->b->c->a plus a->c, unit costs, root a -> {a->b, a->c}
    L = {(0, 1): 1, (1, 2): 1, (2, 0): 1, (0, 2): 1}
    assert packing.min_arborescence(3, 0, L) == (-1, 0, 0)
    # zero-cost Hamiltonian path in K4
    L = {(u, v): 1.0 for u in range(4) for v in range(4) if u != v}
    L[(0, 2)] = L[(2, 1)] = L[(1, 3)] = 0.0
    assert packing.min_arborescence(4, 0, L) == (-1, 2, 0, 1)


def test_min_spanning_tree_matches_brute_force():
    rng = random.Random(7)
    for _ in range(10):
        n = rng.randint(2, 6)
        pairs = random_undirected(rng, n, p=0.8)
        L = {e: rng.random() for e in pairs}
        t = packing.min_spanning_tree(n, L)
        best = min(sum(L[e] for e in tr) for tr in bounds.enumerate_spanning_trees(pairs, n))
        assert abs(sum(L[e] for e in t) - best) < 1e-12


# ------------------------------------------------------------------ MWU
@pytest.mark.parametrize("seed", range(10))
def test_mwu_within_eps_of_edmonds(seed):
    rng = random.Random(900 + seed)
    g = random_digraph(rng, rng.randint(2, 6))
    eps = 0.1
    w, rate, _ = packing.mwu_broadcast(g, 0, eps)
    opt = bounds.edmonds_rate(g, 0)
    assert rate >= (1 - eps) * opt - 1e-9
    assert rate <= opt + 1e-9
    _check_feasible(g[1], {p: x for p, x in w.items()}, directed=True)


@pytest.mark.parametrize("seed", range(6))
def test_mwu_allreduce_within_eps_of_nash_williams(seed):
    rng = random.Random(1300 + seed)
    n = rng.randint(2, 6)
    pairs = random_undirected(rng, n)
    w, rate, _ = packing.mwu_allreduce(pairs, n, 0.1)
    opt = bounds.nash_williams_rate(pairs, n)
    assert (1 - 0.1) * opt - 1e-9 <= rate <= opt + 1e-9
    load = {e: 0.0 for e in pairs}
    for t, x in w.items():
        for e in t:
            load[e] += x
    assert all(load[e] <= pairs[e] + 1e-9 for e in pairs)


def _check_feasible(cap, w, directed):
    load = {e: 0.0 for e in cap}
    for parent, x in w.items():
        for v, p in enumerate(parent):
            if p >= 0:
                load[(p, v)] += x
    assert all(load[e] <= cap[e] + 1e-9 for e in cap)


def test_mwu_dgx1v_rate():
    w, rate, iters = packing.mwu_broadcast(graphs.dgx1v(), 0, 0.1)
    assert 0.9 * 6 <= rate <= 6 + 1e-9
    _check_feasible(graphs.dgx1v()[1], w, True)


# ------------------------------------------------------------------ plans
def _brute_ilp(caps, cand, g):
    """Eqs. 4-7 at grid g by enumerating every z in {0..g}^k: the
    lexicographic optimum (max sum z, fewest trees, smallest maximum depth,
    least total depth) as a key tuple."""
    from itertools import product as iproduct
    best = None
    for z in iproduct(range(g + 1), repeat=len(cand)):
        load = {}
        for zj, (te, _, _) in zip(z, cand):
            for e in te:
                load[e] = load.get(e, 0) + zj
        if any(load[e] > g * caps[e] for e in load):
            continue
        used = [d for zj, (_, d, _) in zip(z, cand) if zj > 0]
        key = (-sum(z), len(used), max(used, default=0), sum(used))
        best = key if best is None or key < best else best
    return best


@pytest.mark.parametrize("seed", range(8))
def test_ilp_refine_tiebreaks_match_brute_force(seed):
    """The ILP's objective and its tie-breaks (R#21) against exhaustive
    enumeration on small candidate sets: random spanning trees of a random
    4-5 GPU graph, grids 1 and 2."""
    rng = random.Random(2600 + seed)
    n = rng.randint(4, 5)
    pairs = random_undirected(rng, n, p=0.8, cmax=2)
    trees = list(bounds.enumerate_spanning_trees(pairs, n))
    rng.shuffle(trees)
    cand = []
    for t in trees[:6]:
        root = packing.tree_centre(list(t), n)
        cand.append((list(t), packing.parent_depth(packing.root_tree(list(t), n, root)), t))
    for g in (1, 2):
        sol, gg, _ = packing.ilp_refine(pairs, cand, 1e9, grids=(g,))
        used = [cand[j][1] for j, _ in sol]
        got = (-sum(w * g for _, w in sol), len(used), max(used, default=0), sum(used))
        assert got == _brute_ilp(pairs, cand, g)


def test_three_gpu_broadcast_plan_is_the_two_chains():
    pin = PINS["three_gpu_broadcast"]
    tri, ids = graphs.induced(graphs.dgx1p(), pin["gpus"])
    plan = packing.plan_broadcast_graph(tri, 0)
    assert plan["rate"] == pin["rate"]
    pos = {g: i for i, g in enumerate(ids)}
    want = set()
    for ring in pin["rings"]:          # ring minus its last hop = a chain
        chain = [pos[g] for g in ring]
        parent = [-1] * 3
        for a, b in zip(chain, chain[1:]):
            parent[b] = a
        want.add(tuple(parent))
    assert {t["parent"] for t in plan["trees"]} == want
    assert all(t["weight"] == 1 for t in plan["trees"])
    # the LP optimum is unique: no other packing of value 2 exists
    assert abs(bounds.brute_broadcast_rate(tri, 0) - 2) < 1e-9


def test_three_gpu_allreduce_plan_relaxes_to_halves():
    tri, _ = graphs.induced(graphs.dgx1p(), [0, 1, 3])
    plan = packing.plan_allreduce_graph(tri)
    assert plan["rate"] == Fraction(3, 2) and plan["grid"] == 2
    assert sorted(t["root"] for t in plan["trees"]) == [0, 1, 2]
    assert all(t["weight"] == Fraction(1, 2) and t["depth"] == 1 for t in plan["trees"])
    # binary level (g=1) only reaches 1.0 (gap 33% > 5%)
    pairs = graphs.undirected_pairs(tri)
    cand = [([(0, 1), (0, 2)], 1, 0), ([(0, 1), (1, 2)], 1, 1), ([(0, 2), (1, 2)], 1, 2)]
    sol, g, ok = packing.ilp_refine(pairs, cand, 1.5, grids=(1,))
    assert sum(w for _, w in sol) == 1 and not ok


def test_dgx1v_plan_six_unit_trees():
    pin = PINS["dgx1v_tree_count_after_ilp"]
    plan = packing.plan_broadcast_graph(graphs.dgx1v(), 0)
    assert len(plan["trees"]) == pin["value"]
    assert all(t["weight"] == 1 for t in plan["trees"])
    assert plan["rate"] == 6
    # 1000 MB over 6 trees: ~166 MB each
    rng = packing.split_bytes(1000 * 10**6, [t["weight"] for t in plan["trees"]])
    assert all(int((hi - lo) / 1e6) == PINS["dgx1v_mb_per_tree_for_1000mb"]["value"] for lo, hi in rng)
    # feasibility and per-port load 1
    _check_feasible(graphs.dgx1v()[1], {t["parent"]: 1.0 for t in plan["trees"]}, True)
    assert packing.link_load(plan, 8, False) == 1


@pytest.mark.slow
def test_dgx1v_allreduce_plan_within_gap():
    g = graphs.dgx1v()
    plan = packing.plan_allreduce_graph(g)
    assert plan["accepted"]
    pairs = graphs.undirected_pairs(g)
    load = {e: Fraction(0) for e in pairs}
    for t in plan["trees"]:
        for e in t["edges"]:
            load[e] += t["weight"]
    assert all(load[e] <= pairs[e] for e in pairs)
    # within 5% of the Nash-Williams optimum 24/7 (R#3)
    assert plan["rate"] >= Fraction(95, 100) * Fraction(24, 7)
    assert plan["opt"] == pytest.approx(24 / 7)


def test_switch_plans_closed_form():
    for m in (1, 2, 3, 5, 8):
        p = packing.plan_switch_allreduce(m)
        assert len(p["trees"]) == m and p["rate"] == Fraction(m, 2)
        for j, t in enumerate(p["trees"]):
            assert t["root"] == j and all(t["parent"][v] == (-1 if v == j else j) for v in range(m))
        # slices of 1/m, exact sums
        S = 1000 * m + 12
        rngs = packing.split_bytes(S, [t["weight"] for t in p["trees"]])
        assert rngs[0][0] == 0 and rngs[-1][1] == S
        G = S // 16
        for j, (lo, hi) in enumerate(rngs):
            assert lo == 16 * (j * G // m)
    for m in (3, 4, 8):
        b = packing.plan_switch_broadcast(m, 1)
        assert b["rate"] == m - 1 and len(b["trees"]) == m - 1
        assert b["rate"] == bounds.edmonds_rate(graphs.complete(m), 1)
        assert packing.link_load(b, m, False) == 1


@pytest.mark.parametrize("S", [0, 1, 15, 16, 17, 1000, 2**20 + 3, 178956970])
def test_split_properties(S):
    for ws in ([1], [1, 1, 1], [Fraction(1, 2)] * 3, [3, 1, 2, 7], [Fraction(1, 16), 1, Fraction(5, 4)]):
        rngs = packing.split_bytes(S, ws)
        assert rngs[0][0] == 0 and rngs[-1][1] == S
        for (a, b), (c, d) in zip(rngs, rngs[1:]):
            assert b == c and a <= b and a % 16 == 0
        W = sum(Fraction(w) for w in ws)
        for (lo, hi), w in zip(rngs[:-1], ws[:-1]):
            assert abs(Fraction(hi - lo) - Fraction(S) * Fraction(w) / W) < 32


# ------------------------------------------------------------------ NEXT-4
def test_multiserver_plan_structure_3_plus_5():
    # the paper's 2 x DGX-1V experiment allocates 3 + 5 GPUs;
    # here: DGX-1V GPUs {0,1,3} on server 0 and {2,4,5,6,7} on server 1
    from oracle import collectives as C
    g = graphs.dgx1v()
    servers = [[0, 1, 3], [2, 4, 5, 6, 7]]
    # cross-server links are not NVLink: drop GPU-GPU links between servers
    cap = {(u, v): c for (u, v), c in g[1].items()
           if any(u in s and v in s for s in servers)}
    gg = (8, cap)
    plan = packing.plan_multiserver_allreduce(gg, servers)
    K = plan["partitions"]
    assert len(plan["trees"]) == K * len(servers)           # n one-hop cross trees per partition
    for t in plan["trees"]:
        assert t["parent"].count(-1) == 1 and t["root"] in servers[t["server"]]
        cross = [(u, v) for (u, v) in t["edges"] if not any(u in s and v in s for s in servers)]
        assert len(cross) == len(servers) - 1                # one hop between local roots
        assert len(t["edges"]) == 7                          # spanning tree of 8 GPUs
    for p in range(K):
        roots = {t["root"] for t in plan["trees"] if t["partition"] == p}
        assert len(roots) == len(servers)                    # one root per server per partition
    # distinct server-local roots across partitions where the server has room
    for s, ids in enumerate(servers):
        rs = [t["root"] for t in plan["trees"] if t["server"] == s]
        assert len(set(rs)) == min(K, len(ids))
    # integer AllReduce along it is exact (any tree order)
    sends = synth.inputs(7, 8, 999, "i32")
    assert np.array_equal(C.allreduce(plan, sends, "i32", "sum"), C.naive_reduce(sends, "i32", "sum"))


def test_multiserver_single_gpu_servers_is_the_dgx2_onehop_plan():
    # n servers of one GPU each: phase 1 and 3 vanish and phase 2 is exactly
    # the m one-hop trees of P:440-442
    m = 5
    plan = packing.plan_multiserver_allreduce((m, {}), [[v] for v in range(m)])
    ref = packing.plan_switch_allreduce(m)
    assert [t["parent"] for t in plan["trees"]] == [t["parent"] for t in ref["trees"]]
