"""Pins for oracle/model.py: the chunk-pipelining model and the
bytes every plan moves.  SURVEY 8(c-5) rows "Pipeline" and
"Bytes moved"."""
from fractions import Fraction

import pytest

from oracle import graphs, model, packing


def chain(n):
    return tuple(-1 if v == 0 else v - 1 for v in range(n))


def test_paper_four_gpu_example_two_chunks_save_a_third():
    """"Splitting data into two chunks reduces transfer time by a
    third when compared to a setting with no chunking" (four GPUs)."""
    one = model.pipeline_makespan(chain(4), 1)
    two = model.pipeline_makespan(chain(4), 2)
    assert one == 3 and two == 2
    assert (one - two) / one == Fraction(1, 3)


@pytest.mark.parametrize("hops", range(1, 8))
def test_simulation_matches_the_closed_form_on_chains(hops):
    for c in range(1, 17):
        assert model.pipeline_makespan(chain(hops + 1), c) == model.chain_time(c, hops)


def test_star_gains_nothing_from_chunking_and_deeper_trees_gain_more():
    star = tuple(-1 if v == 0 else 0 for v in range(8))
    assert all(model.pipeline_makespan(star, c) == 1 for c in (1, 2, 7, 64))
    # more chunks never hurt in the model (no per-chunk overhead), and the
    # limit is one link time
    prev = None
    for c in (1, 2, 4, 8, 64, 512):
        t = model.pipeline_makespan(chain(6), c)
        assert prev is None or t < prev
        prev = t
    assert model.pipeline_makespan(chain(6), 512) - 1 == Fraction(4, 512)


def test_branching_trees_follow_their_depth():
    """Links run concurrently, so a tree pipelines like its deepest path: the
    DGX-1V Broadcast trees (depth 4-5) included."""
    plan = packing.plan_broadcast_graph(graphs.dgx1v(), 0)
    for t in plan["trees"]:
        depth = packing.parent_depth(t["parent"])
        for c in (1, 3, 16):
            assert model.pipeline_makespan(t["parent"], c) == model.chain_time(c, depth)


@pytest.mark.parametrize("m", [2, 3, 5, 8])
def test_onehop_allreduce_moves_2_m_minus_1_over_m_per_gpu(m):
    """2(N-1)/N of the data per process; exactly, with the 16-byte
    split, GPU v sends S + (m - 2) * |slice v| bytes and receives as much."""
    plan = packing.plan_switch_allreduce(m)
    for S in (16 * m * 1000, 16 * m * 1000 + 5, 1 << 20):
        lb = model.link_bytes(plan, m, S, True)
        rng = packing.split_bytes(S, [t["weight"] for t in plan["trees"]])
        for v in range(m):
            eg = sum(b for (u, _), b in lb.items() if u == v)
            ing = sum(b for (_, w), b in lb.items() if w == v)
            sv = rng[v][1] - rng[v][0]
            assert eg == ing == S + (m - 2) * sv
            assert abs(Fraction(eg) - Fraction(2 * (m - 1) * S, m)) <= 16 * (m - 2) + 16


@pytest.mark.parametrize("name", ["switch8", "dgx1v", "dgx1p", "tri"])
def test_total_bytes_match_the_message_bound(name):
    """Any plan of spanning trees moves (m-1) S for Broadcast and 2 (m-1) S
    for AllReduce in total (N-1 edges per tree, both directions for
    AllReduce), and every non-root GPU receives exactly S in a Broadcast."""
    if name == "switch8":
        m, bplan, aplan = 8, packing.plan_switch_broadcast(8, 3), packing.plan_switch_allreduce(8)
        root = 3
    elif name == "tri":
        g, _ = graphs.induced(graphs.dgx1p(), [0, 1, 3])
        m, root = 3, 0
        bplan, aplan = packing.plan_broadcast_graph(g, 0), packing.plan_allreduce_graph(g)
    else:
        g = graphs.dgx1v() if name == "dgx1v" else graphs.dgx1p()
        m, root = 8, 0
        bplan = packing.plan_broadcast_graph(g, 0)
        aplan = packing.plan_switch_allreduce(8) if name == "dgx1p" else None
    S = 1000003
    lb = model.link_bytes(bplan, m, S, False)
    assert sum(lb.values()) == (m - 1) * S
    for v in range(m):
        ing = sum(b for (_, w), b in lb.items() if w == v)
        assert ing == (0 if v == root else S)
    if aplan is not None:
        la = model.link_bytes(aplan, m, S, True)
        assert sum(la.values()) == 2 * (m - 1) * S


def test_dgx1v_broadcast_respects_link_capacity_per_byte():
    """6 unit trees on 24 link units: no link unit carries more than S/6 (+ the
    16-byte grain), i.e. the per-port load L = 1 of SURVEY 8(d) config 2."""
    g = graphs.dgx1v()
    plan = packing.plan_broadcast_graph(g, 0)
    S = 6 * 10**6 + 7
    lb = model.link_bytes(plan, 8, S, False)
    cap = g[1]
    for (u, v), b in lb.items():
        assert b <= cap[(u, v)] * (S // 6 + 16)


def test_hybrid_split_equalises_the_two_transfer_times():
    """Eq. 8: the split satisfies its defining objective
    T_PCIe + T_dpa = T_NVL exactly (checked as times, not by retyping the
    closed form), conserves D_total, reduces to the bandwidth-proportional
    split at T_dpa = 0, and clamps (R#31) when T_dpa exceeds T_NVL of the
    whole buffer."""
    from fractions import Fraction
    from oracle import model
    for D, bp, bn, t in ((10**9, 32 * 10**9, 150 * 10**9, Fraction(1, 10**3)),
                         (3 * 10**8, 16 * 10**9, 50 * 10**9, Fraction(5, 10**4)),
                         (12345678, 25 * 10**9, 300 * 10**9, Fraction(0))):
        dp, dn = model.hybrid_split(D, bp, bn, t)
        assert dp + dn == D and 0 <= dp <= D
        assert dp / bp + t == dn / bn                      # T_PCIe + T_dpa = T_NVL
        if t == 0:
            assert dp * bn == dn * bp                      # proportional to bandwidth
    dp, dn = model.hybrid_split(10**6, 32 * 10**9, 150 * 10**9, Fraction(1))   # T_dpa >> T_NVL
    assert dp == 0 and dn == 10**6
