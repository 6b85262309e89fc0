"""Pins for oracle/graphs.py: the DGX-1 reconstruction (R#17) against every
consequence the paper's text states (tests/golden/paper_pins.json)."""
import json
import os
from itertools import permutations

import pytest

from oracle import graphs

PINS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_pins.json")))


def _deg(g, v):
    n, cap = g
    return sum(c for (u, w), c in cap.items() if u == v)


def test_port_counts():
    # P100 has 4 NVLink ports, V100 6 (P:59 gen1 / gen2): every port used.
    assert all(_deg(graphs.dgx1p(), v) == 4 for v in range(8))
    assert all(_deg(graphs.dgx1v(), v) == 6 for v in range(8))
    assert sum(graphs.dgx1v()[1].values()) == 2 * 24


def test_missing_link_1_4():
    u, v = PINS["dgx1p_missing_link"]["pair"]
    for g in (graphs.dgx1p(), graphs.dgx1v()):
        assert (u, v) not in g[1] and (v, u) not in g[1]


def test_ring_2_6_7_3_and_no_diagonals():
    ring = PINS["dgx1v_ring_2367"]["ring"]
    sub, ids = graphs.induced(graphs.dgx1v(), ring)
    pos = {g: i for i, g in enumerate(ids)}
    for a, b in zip(ring, ring[1:] + ring[:1]):
        assert (pos[a], pos[b]) in sub[1]
    assert (pos[2], pos[7]) not in sub[1] and (pos[3], pos[6]) not in sub[1]


def _ham_cycles(g):
    n, cap = g
    out = []
    for perm in permutations(range(1, n)):
        cyc = (0,) + perm
        if all((cyc[i], cyc[(i + 1) % n]) in cap for i in range(n)):
            out.append(cyc)
    return out


def test_no_nvlink_ring_1_4_5_6():
    sub, _ = graphs.induced(graphs.dgx1v(), PINS["dgx1v_no_ring_1456"]["gpus"])
    assert graphs.is_connected(sub)
    assert _ham_cycles(sub) == []


def test_6gpu_unused_links():
    pin = PINS["dgx1p_6gpu_unused_links"]
    sub, ids = graphs.induced(graphs.dgx1p(), pin["gpus"])
    links = {(ids[u], ids[v]) for (u, v) in sub[1] if u < v}
    unused = {tuple(sorted(p)) for p in pin["unused"]}
    assert unused <= links
    assert len(links) == 9
    # some Hamiltonian ring uses exactly the other 6 links
    found = False
    for cyc in _ham_cycles(sub):
        used = {tuple(sorted((ids[cyc[i]], ids[cyc[(i + 1) % 6]]))) for i in range(6)}
        if links - used == unused:
            found = True
    assert found


def test_three_gpu_allocation_fully_connected():
    sub, _ = graphs.induced(graphs.dgx1p(), PINS["three_gpu_broadcast"]["gpus"])
    assert sub[1] == {(u, v): 1 for u in range(3) for v in range(3) if u != v}


@pytest.mark.slow
def test_unique_allocation_bins_46_14():
    pin = PINS["unique_allocations"]
    v = graphs.unique_allocations(graphs.dgx1v())
    p = graphs.unique_allocations(graphs.dgx1p())
    assert sum(v.values()) == pin["dgx1v"]
    assert sum(p.values()) == pin["dgx1p"]


def test_induced_identity_and_undirected():
    g = graphs.dgx1v()
    sub, ids = graphs.induced(g, range(8))
    assert sub == g and ids == list(range(8))
    pairs = graphs.undirected_pairs(g)
    assert len(pairs) == 16 and sum(pairs.values()) == 24
    with pytest.raises(ValueError):
        graphs.undirected_pairs((2, {(0, 1): 1}))
