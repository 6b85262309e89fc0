"""GPU parity of work stealing (DESIGN 2b "Work stealing"): CTAs whose own
channel has handed out every chunk join other channels of the launch.

Chunks of 36-40 KiB (above the register path's 32 KiB, so the TMA pipeline
runs) give every channel many more chunks than CTAs, so joins happen at test
sizes; `last_steal_channels` proves the launch had stealing on.  Results must stay bit-exact against the oracle (a joined chunk
is combined by the same channel code in the same operand order).
"""
import numpy as np
import pytest

import synth
from oracle import collectives as OC
from oracle import graphs as OG
from test_gpu_parity import (assert_bitwise, make_comms, oracle_plan_from_json, run_allreduce,
                             sentinel, to_dev, to_host)

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1910_04940_b200 as B
    return B


@pytest.mark.parametrize("per_rank", [False, True])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_steal_dgx1v_allreduce_bitexact(B, dtype, per_rank):
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=36864,
                       launch_per_rank=int(per_rank))
    count = (3 << 20) + 7
    sends = synth.inputs(77, 8, count, dtype)
    got = run_allreduce(B, comms, sends, dtype, "sum")
    assert comms[0].stats()["last_steal_channels"] > 0
    want = OC.allreduce(oracle_plan_from_json(comms[0].plan(True, 0, count, dtype)), sends, dtype, "sum")
    for x in got:
        assert_bitwise(x, want)
    # the same call again (counters were reset by the last CTA; epochs advance)
    got = run_allreduce(B, comms, sends, dtype, "sum")
    for x in got:
        assert_bitwise(x, want)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("root", [0, 7])
def test_steal_dgx1v_broadcast_bitexact(B, root):
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=40960)
    count = (4 << 20) + 5
    send = synth.rank_input(9, root, count, "f32")
    recv = [sentinel(count, "f32") for _ in range(8)]
    src = to_dev(send, "f32")
    for r, c in enumerate(comms):
        c.broadcast(src if r == root else None, recv[r], root=root)
    torch.cuda.synchronize()
    assert comms[0].stats()["last_steal_channels"] > 0
    for x in recv:
        assert_bitwise(to_host(x, "f32"), send)
    for c in comms:
        c.destroy()


def test_steal_int_exact_under_any_join_order(B):
    """int32 SUM is exact: any chunk-to-CTA assignment gives the naive sum."""
    tri, _ = OG.induced(OG.dgx1v(), [0, 1, 3, 4, 5, 7])
    comms = make_comms(B, 6, graph=B.Graph.from_pairs(6, tri[1]), chunk_bytes=36864)
    count = (1 << 20) + 17
    sends = synth.inputs(5, 6, count, "i32")
    got = run_allreduce(B, comms, sends, "i32", "sum")
    assert comms[0].stats()["last_steal_channels"] > 0
    want = OC.naive_reduce(sends, "i32", "sum")
    for x in got:
        assert np.array_equal(x, want)
    for c in comms:
        c.destroy()


def test_steal_off_same_bits(B, monkeypatch):
    """BLINK_STEAL=0 is read once per process; compare against a launch whose
    channels cannot be joined (chunks <= 3 x CTAs) instead: same bits."""
    g = OG.dgx1v()
    count = (1 << 19) + 3
    sends = synth.inputs(12, 8, count, "f32")
    a = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=36864)
    got_a = run_allreduce(B, a, sends, "f32", "sum")
    assert a[0].stats()["last_steal_channels"] > 0
    plan_a = a[0].plan(True, 0, count, "f32")
    for c in a:
        c.destroy()
    b = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=1 << 20)
    got_b = run_allreduce(B, b, sends, "f32", "sum")
    assert b[0].stats()["last_steal_channels"] == 0
    assert [t["parent"] for t in plan_a["trees"]] == [t["parent"] for t in b[0].plan(True, 0, count, "f32")["trees"]]
    for c in b:
        c.destroy()
    for x, y in zip(got_a, got_b):
        assert_bitwise(x, y)
