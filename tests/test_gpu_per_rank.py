"""GPU parity for per-rank launches (cfg.launch_per_rank = 1).

Every virtual rank runs in its own launch on its own stream, so the
cross-launch protocol of the one-process-per-GPU path runs for real and
concurrently on one B200: entry handshakes, per-chunk flags between launches,
exit waits.  Separate processes on one GPU time-slice instead
of running concurrently, so this is where that protocol is exercised and timed
on the 1-GPU box.  Expected values come only from oracle/ (same rules as
test_gpu_parity.py).
"""
import numpy as np
import pytest

import synth
from oracle import collectives as OC
from oracle import graphs as OG
from oracle import packing as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import (B, assert_bitwise, oracle_plan_from_json, run_allreduce,  # noqa: E402,F401
                             sentinel, to_dev, to_host)


def per_rank_comms(B, m, graph=None, **cfg):
    cfg.setdefault("timeout_s", 20.0)
    return B.init_all([0] * m, graph=graph, cfg=B.config(launch_per_rank=1, **cfg))


@pytest.mark.parametrize("m", [2, 3, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_per_rank_onehop_allreduce(B, m, dtype):
    count = 4096 * m + 13
    sends = synth.inputs(130 + m, m, count, dtype)
    comms = per_rank_comms(B, m, chunk_bytes=4096)
    for op in ("sum", "max"):
        got = run_allreduce(B, comms, sends, dtype, op)
        want = OC.allreduce(OP.plan_switch_allreduce(m), sends, dtype, op)
        for g in got:
            assert_bitwise(g, want)
    # one launch per rank, each with its own CTAs
    assert comms[0].stats()["launches"] == 2
    assert comms[0].stats()["last_ctas"] <= 148 // m
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("count", [1, 1000, (1 << 20) + 5])
def test_per_rank_dgx1v_broadcast_multihop(B, count):
    g = OG.dgx1v()
    comms = per_rank_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]))
    root = 3
    send = synth.rank_input(2, root, count, "f32")
    dsend = to_dev(send, "f32")
    recvs = [sentinel(count, "f32") for _ in range(8)]
    for r, c in enumerate(comms):
        c.broadcast(dsend if r == root else None, recvs[r], root=root, count=count, dtype="f32")
    torch.cuda.synchronize()
    for x in recvs:
        assert_bitwise(x.cpu().numpy(), send)
    for c in comms:
        c.destroy()


def test_per_rank_dgx1v_allreduce_tree_order(B):
    g = OG.dgx1v()
    comms = per_rank_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=16384)
    count = 200003
    sends = synth.inputs(21, 8, count, "f32")
    got = run_allreduce(B, comms, sends, "f32", "sum")
    plan = oracle_plan_from_json(comms[0].plan(True, 0, count, "f32"))
    want = OC.allreduce(plan, sends, "f32", "sum")
    for x in got:
        assert_bitwise(x, want)
    ints = synth.inputs(22, 8, count, "i32")
    for x in run_allreduce(B, comms, ints, "i32", "sum"):
        assert_bitwise(x, OC.naive_reduce(ints, "i32", "sum"))
    for c in comms:
        c.destroy()


def test_per_rank_block_collectives_and_gather(B):
    m, B_ = 8, 33333
    comms = per_rank_comms(B, m, chunk_bytes=8192)
    sends = synth.inputs(140, m, m * B_, "f32")
    ds = [to_dev(s, "f32") for s in sends]
    rs = [sentinel(B_, "f32") for _ in range(m)]
    for r, c in enumerate(comms):
        c.reduce_scatter(ds[r], rs[r], op="sum", recvcount=B_, dtype="f32")
    torch.cuda.synchronize()
    want = OC.reduce_scatter(sends, "f32", "sum")
    for r in range(m):
        assert_bitwise(rs[r].cpu().numpy(), want[r])
    ag = [sentinel(m * B_, "f32") for _ in range(m)]
    for r, c in enumerate(comms):
        c.allgather(rs[r], ag[r], sendcount=B_, dtype="f32")
    torch.cuda.synchronize()
    for r in range(m):
        assert_bitwise(ag[r].cpu().numpy(), OC.allgather(want))
    root = 5
    gat = sentinel(m * B_, "f32")
    for r, c in enumerate(comms):
        c.gather(rs[r], gat if r == root else None, root=root, sendcount=B_, dtype="f32")
    torch.cuda.synchronize()
    assert_bitwise(gat.cpu().numpy(), OC.allgather(want))
    for c in comms:
        c.destroy()


def test_per_rank_streams_back_to_back_and_graph_replay(B):
    """Each rank on its own user stream; six calls without a host sync; then a
    captured call replayed with new inputs (epochs live on the device)."""
    m, count = 8, 65537
    comms = per_rank_comms(B, m, chunk_bytes=8192)
    streams = [torch.cuda.Stream() for _ in range(m)]
    sends = synth.inputs(150, m, count, "f32")
    dsend = [to_dev(s, "f32") for s in sends]
    outs = [[torch.empty_like(d) for d in dsend] for _ in range(6)]
    torch.cuda.synchronize()
    for k in range(6):
        for r, c in enumerate(comms):
            c.allreduce(dsend[r], outs[k][r], op="sum", stream=streams[r])
    torch.cuda.synchronize()
    want = OC.naive_reduce(sends, "f32", "sum")
    for k in range(6):
        for x in outs[k]:
            assert_bitwise(x.cpu().numpy(), want)
    drecv = [torch.empty_like(d) for d in dsend]
    for r, c in enumerate(comms):
        c.allreduce(dsend[r], drecv[r])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r, c in enumerate(comms):
            c.allreduce(dsend[r], drecv[r])
    for it in range(3):
        sends = synth.inputs(160 + it, m, count, "f32")
        for d, s in zip(dsend, sends):
            d.copy_(torch.from_numpy(s))
        g.replay()
        torch.cuda.synchronize()
        want = OC.naive_reduce(sends, "f32", "sum")
        for x in drecv:
            assert_bitwise(x.cpu().numpy(), want)
    for c in comms:
        c.destroy()


def test_per_rank_large_sampled(B):
    """8 x 64 MiB per rank: every chunk of every tree crosses launches."""
    m, count = 8, 16 << 20
    comms = per_rank_comms(B, m)
    xs = [synth.device_input(3, r, count, "f32") for r in range(m)]
    ys = [torch.empty_like(x) for x in xs]
    for r, c in enumerate(comms):
        c.allreduce(xs[r], ys[r])
    torch.cuda.synchronize()
    rng = np.random.default_rng(7)
    idx = np.unique(np.concatenate([rng.integers(0, count, 20000), np.arange(count - 64, count)]))
    ti = torch.from_numpy(idx).cuda()
    sends = [x[ti].cpu().numpy() for x in xs]
    want = OC.naive_reduce(sends, "f32", "sum")
    for y in ys:
        assert_bitwise(y[ti].cpu().numpy(), want)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("graph_name", ["switch", "dgx1v"])
def test_per_rank_chunking_agrees_across_ranks(B, graph_name):
    """A chunk's flags name the same bytes on every rank, so every launch
    group (rank) must chunk a tree identically, whatever channels it runs
    (the root of 7 two-level trees vs an inner node with one forward channel)."""
    graph = None if graph_name == "switch" else B.Graph.from_pairs(8, OG.dgx1v()[1])
    comms = per_rank_comms(B, 8, graph=graph)
    for is_ar in (False, True):
        for count in (1 << 20, (16 << 20) + 3, 64 << 20):
            views = [c.plan(is_ar, 0, count) for c in comms]
            key = [[(t["lo"], t["hi"], t["chunk"], t["nchunks"]) for t in p["trees"]] for p in views]
            assert all(k == key[0] for k in key), (is_ar, count)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("graph_name", ["switch", "dgx1v"])
def test_per_rank_large_broadcast_every_byte(B, graph_name):
    graph = None if graph_name == "switch" else B.Graph.from_pairs(8, OG.dgx1v()[1])
    comms = per_rank_comms(B, 8, graph=graph)
    count, root = (16 << 20) + 5, 6
    x = synth.device_input(2, root, count, "f32")
    ys = [torch.zeros_like(x) for _ in range(8)]
    for r, c in enumerate(comms):
        c.broadcast(x if r == root else None, ys[r], root=root)
    torch.cuda.synchronize()
    for y in ys:
        assert torch.equal(y.view(torch.int32), x.view(torch.int32))
    for c in comms:
        c.destroy()


def test_per_rank_large_multilevel_allreduce_int_exact(B):
    g = OG.dgx1v()
    comms = per_rank_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]))
    count = (8 << 20) + 7
    xs = [synth.device_input(5, r, count, "i32") for r in range(8)]
    ys = [torch.empty_like(x) for x in xs]
    for r, c in enumerate(comms):
        c.allreduce(xs[r], ys[r])
    torch.cuda.synchronize()
    want = xs[0].clone()
    for x in xs[1:]:
        want += x   # int32 wraparound sum: exact under any order (definition, SURVEY c-1)
    for y in ys:
        assert torch.equal(y, want)
    for c in comms:
        c.destroy()


def test_per_rank_miad_autotune(B):
    """NEXT-2 with per-rank launches (the multi-process protocol's kernels):
    MIAD moves the chunk size across calls, every rank's launch chunks each
    call identically, and every call stays bit-exact."""
    m, count = 4, (2 << 20) + 7
    comms = per_rank_comms(B, m, autotune=1)
    sends = synth.inputs(121, m, count, "f32")
    want = OC.naive_reduce(sends, "f32", "sum")
    ds = [to_dev(s, "f32") for s in sends]
    out = [torch.empty_like(d) for d in ds]
    chunks = []
    for it in range(14):
        for r, c in enumerate(comms):
            c.allreduce(ds[r], out[r])
        torch.cuda.synchronize()
        per = {c.stats()["last_chunk_bytes"] for c in comms}
        assert len(per) == 1, per
        chunks.append(per.pop())
        for x in out:
            assert_bitwise(x.cpu().numpy(), want)
    assert len(set(chunks)) >= 2, chunks
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("dtype", ["f32", "i32"])
def test_per_rank_link_graph_allgather_and_gather(B, dtype):
    """NEXT-3 on DGX-1V with per-rank launches: relays wait for their chain
    parent's per-chunk flags across launches, exit waits cover every block a
    rank receives."""
    g = OG.dgx1v()
    comms = per_rank_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=8192)
    B_ = 70001
    sends = synth.inputs(170, 8, B_, dtype)
    ds = [to_dev(s, dtype) for s in sends]
    outs = [sentinel(8 * B_, dtype) for _ in range(8)]
    for r, c in enumerate(comms):
        c.allgather(ds[r], outs[r], sendcount=B_, dtype=dtype)
    torch.cuda.synchronize()
    for o in outs:
        assert_bitwise(to_host(o, dtype), OC.allgather(sends))
    for root in (0, 6):
        out = sentinel(8 * B_, dtype)
        for r, c in enumerate(comms):
            c.gather(ds[r], out if r == root else None, root=root, sendcount=B_, dtype=dtype)
        torch.cuda.synchronize()
        assert_bitwise(to_host(out, dtype), OC.gather(sends, root)[root])
    # ReduceScatter: inner ranks relay partials and ack their children
    rs = synth.inputs(171, 8, 8 * B_, dtype)
    dr = [to_dev(s, dtype) for s in rs]
    outs = [sentinel(B_, dtype) for _ in range(8)]
    for r, c in enumerate(comms):
        c.reduce_scatter(dr[r], outs[r], op="max", recvcount=B_, dtype=dtype)
    torch.cuda.synchronize()
    want = OC.reduce_scatter(rs, dtype, "max")
    for r in range(8):
        assert_bitwise(to_host(outs[r], dtype), want[r])
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("warm", [1, 0])
@pytest.mark.parametrize("per_rank", [0, 1])
def test_miad_calls_inside_a_cuda_graph_capture(B, per_rank, warm):
    """With cfg.autotune, a call captured into a CUDA graph takes the chunk
    the eager calls tuned so far without timing it (the static table's when
    the capture is the first call, whose tables are then built outside the
    capture); replays are bit-exact, and eager calls afterwards still tune."""
    m, count = 4, (1 << 20) + 3
    comms = B.init_all([0] * m, cfg=B.config(timeout_s=20.0, autotune=1, launch_per_rank=per_rank))
    sends = synth.inputs(122, m, count, "f32")
    want = OC.naive_reduce(sends, "f32", "sum")
    ds = [to_dev(s, "f32") for s in sends]
    out = [torch.empty_like(d) for d in ds]
    for _ in range(3 if warm else 0):  # eager warm-up (tuning)
        for r, c in enumerate(comms):
            c.allreduce(ds[r], out[r])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=s):
        for r, c in enumerate(comms):
            c.allreduce(ds[r], out[r], stream=torch.cuda.current_stream())
    for _ in range(3):
        for o in out:
            o.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        for o in out:
            assert_bitwise(o.cpu().numpy(), want)
    for r, c in enumerate(comms):
        c.allreduce(ds[r], out[r])
    torch.cuda.synchronize()
    for o in out:
        assert_bitwise(o.cpu().numpy(), want)
    for c in comms:
        c.destroy()
