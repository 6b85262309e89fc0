"""GPU parity: the CUDA path (through the C ABI) against the oracle.

All ranks are virtual ranks on cuda:0 (the GPU box has one B200): their
buffers live in one HBM and one cooperative launch runs every rank's channels,
exactly the kernels and tables the multi-GPU path runs (DESIGN.md
"Virtual ranks").  Expected values come only from oracle/ on the same seeded
inputs:
  * Broadcast: bitwise copy of the root's send (definition).
  * AllReduce on one-hop / unique plans: bit-exact vs the oracle's OWN plan.
  * AllReduce on other multi-level plans: the library's plan is first checked
    against the oracle's invariants (tests/test_capi_cpu.py), then the GPU
    result must be bit-exact vs the oracle's tree-order evaluation of that
    plan and within rtol * sum|x| of the naive-order sum (R#20).
  * int32 and MIN/MAX: exact vs the oracle under any plan.
Receive buffers start as 0xFF sentinels so unwritten bytes show up.
"""
import numpy as np
import pytest

import synth
from oracle import collectives as OC
from oracle import graphs as OG
from oracle import packing as OP

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TORCH_DT = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32}
NP_VIEW = {"f32": np.float32, "bf16": np.int16, "i32": np.int32}


@pytest.fixture(scope="module")
def B():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1910_04940_b200 as B
    return B


def to_dev(arr, dtype):
    a = np.ascontiguousarray(arr)
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
    return torch.from_numpy(a.copy()).cuda()


def to_host(t, dtype):
    if dtype == "bf16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def sentinel(count, dtype, offset=0):
    es = OC.ESIZE[dtype]
    raw = torch.full((count * es + offset + 16,), 0xFF, dtype=torch.uint8, device="cuda")
    return raw[offset:offset + count * es].view(TORCH_DT[dtype]) if offset % es == 0 else raw


def oracle_plan_from_json(p):
    from fractions import Fraction
    return dict(trees=[dict(parent=tuple(t["parent"]), root=t["root"],
                            weight=Fraction(*t["weight"])) for t in p["trees"]])


def run_allreduce(B, comms, sends, dtype, op, inplace=False):
    m = len(comms)
    count = len(sends[0])
    dsend = [to_dev(s, dtype) for s in sends]
    drecv = dsend if inplace else [sentinel(count, dtype) for _ in range(m)]
    for r, c in enumerate(comms):
        c.allreduce(dsend[r], drecv[r], op=op, count=count, dtype=dtype)
    torch.cuda.synchronize()
    return [to_host(x, dtype) for x in drecv]


def bits(a):
    a = np.asarray(a)
    return a.view(np.uint16) if a.dtype.itemsize == 2 else a.view(np.uint32)


def assert_bitwise(got, want):
    gb, wb = bits(got), bits(want)
    bad = np.nonzero(gb != wb)[0]
    assert bad.size == 0, f"{bad.size} mismatches, first at {bad[:5]}: got {got[bad[:5]]} want {want[bad[:5]]}"


def make_comms(B, m, graph=None, **cfg):
    cfg.setdefault("timeout_s", 20.0)
    return B.init_all([0] * m, graph=graph, cfg=B.config(**cfg))


# ----------------------------------------------------------------- config 3/4: switch one-hop
@pytest.mark.parametrize("m", [2, 3, 5, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("op", ["sum", "min", "max", "prod", "avg"])
def test_onehop_allreduce_bitexact(B, m, dtype, op):
    count = 2048 * m + 13          # several tiles + a ragged, sub-16-byte tail
    sends = synth.inputs(30 + m, m, count, dtype)
    if op == "prod" and dtype == "i32":
        sends = [(s % 5 - 2).astype(np.int32) for s in sends]
    comms = make_comms(B, m, chunk_bytes=4096)
    got = run_allreduce(B, comms, sends, dtype, op)
    want = OC.allreduce(OP.plan_switch_allreduce(m), sends, dtype, op)
    for g in got:
        assert_bitwise(g, want)
    # one-hop tree order = naive left-to-right order (R#12)
    assert_bitwise(want, OC.naive_reduce(sends, dtype, op))
    for c in comms:
        c.destroy()


def test_onehop_edge_values_f32(B):
    m, count = 6, 4099
    sends = [synth.edge_case_f32(4, r, count) for r in range(m)]
    comms = make_comms(B, m)
    for op in ("sum", "min", "max"):
        got = run_allreduce(B, comms, sends, "f32", op)
        want = OC.allreduce(OP.plan_switch_allreduce(m), sends, "f32", op)
        for g in got:
            assert_bitwise(g, want)


# Multi-level trees with the edge-case set (+-0, subnormals, +-1e30
# cancellation pairs, NaN-free): the register path (8 KiB chunks), and the TMA
# pipeline with work stealing (36 KiB chunks, 3 MiB calls), both bit-exact
# against the oracle's evaluation of the library's own plan in tree order.
@pytest.mark.parametrize("chunk,count", [(8192, 120003), (36864, (3 << 18) + 5)])
def test_multilevel_edge_values_f32(B, chunk, count):
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=chunk, shallow_max_bytes=0,
                       ll_max_bytes=0)
    sends = [synth.edge_case_f32(6, r, count) for r in range(8)]
    for op in ("sum", "min", "max"):
        got = run_allreduce(B, comms, sends, "f32", op)
        want = OC.allreduce(oracle_plan_from_json(comms[0].plan(True, 0, count, "f32")), sends, "f32", op)
        for x in got:
            assert_bitwise(x, want)
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("count", [0, 1, 2, 3, 4, 5, 7, 8, 9, 31, 33, 1000])
def test_tiny_and_ragged_counts(B, count):
    m = 8
    comms = make_comms(B, m)
    for dtype in ("f32", "bf16"):
        sends = synth.inputs(50, m, count, dtype)
        got = run_allreduce(B, comms, sends, dtype, "sum")
        if count:
            want = OC.allreduce(OP.plan_switch_allreduce(m), sends, dtype, "sum")
            for g in got:
                assert_bitwise(g, want)


def test_inplace_and_misaligned(B):
    m, count = 4, 10007
    comms = make_comms(B, m)
    sends = synth.inputs(60, m, count, "f32")
    got = run_allreduce(B, comms, sends, "f32", "sum", inplace=True)
    want = OC.allreduce(OP.plan_switch_allreduce(m), sends, "f32", "sum")
    for g in got:
        assert_bitwise(g, want)
    # misaligned (4-byte offset) views -> scalar path
    dsend, drecv = [], []
    for s in sends:
        buf = torch.empty(count + 1, dtype=torch.float32, device="cuda")
        buf[1:] = torch.from_numpy(s).cuda()
        dsend.append(buf[1:])
        r = torch.full((count + 3,), float("nan"), device="cuda")
        drecv.append(r[3:])
    for r, c in enumerate(comms):
        c.allreduce(dsend[r], drecv[r], op="sum")
    torch.cuda.synchronize()
    for x in drecv:
        assert_bitwise(x.cpu().numpy(), want)


def test_single_rank_is_a_copy(B):
    comms = make_comms(B, 1)
    s = synth.inputs(70, 1, 12345, "bf16")
    got = run_allreduce(B, comms, s, "bf16", "sum")
    assert_bitwise(got[0], s[0])


# ----------------------------------------------------------------- config 1: paper's 3-GPU example
def triangle():
    tri, _ = OG.induced(OG.dgx1p(), [0, 1, 3])
    return tri


def test_config1_three_gpu_allreduce_and_broadcast(B):
    tri = triangle()
    comms = make_comms(B, 3, graph=B.Graph.from_pairs(3, tri[1]))
    count = 262144                    # 1 MiB fp32 (BASELINE configs[0])
    sends = synth.inputs(1, 3, count, "f32")
    got = run_allreduce(B, comms, sends, "f32", "sum")
    # the oracle's own plan (unique LP optimum: three 1/2-weight paths)
    want = OC.allreduce(OP.plan_allreduce_graph(tri), sends, "f32", "sum")
    for g in got:
        assert_bitwise(g, want)
    isends = synth.inputs(1, 3, count, "i32")
    got = run_allreduce(B, comms, isends, "i32", "sum")
    iwant = OC.naive_reduce(isends, "i32", "sum")
    for g in got:
        assert_bitwise(g, iwant)
    # Broadcast from GPU 0 along the two chains
    dsend = to_dev(sends[0], "f32")
    recvs = [sentinel(count, "f32") for _ in range(3)]
    for r, c in enumerate(comms):
        c.broadcast(dsend if r == 0 else None, recvs[r], root=0, count=count, dtype="f32")
    torch.cuda.synchronize()
    for x in recvs:
        assert_bitwise(x.cpu().numpy(), sends[0])
    assert comms[0].plan(False, 0, count)["rate"] == [2, 1]


# ----------------------------------------------------------------- config 2: emulated DGX-1V
@pytest.mark.parametrize("root", [0, 3, 7])
@pytest.mark.parametrize("count", [1, 257, 1 << 20, (1 << 22) + 5])
def test_config2_dgx1v_broadcast(B, root, count):
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]))
    dtype = "f32"
    send = synth.rank_input(2, root, count, dtype)
    dsend = to_dev(send, dtype)
    recvs = [sentinel(count, dtype) for _ in range(8)]
    for r, c in enumerate(comms):
        c.broadcast(dsend if r == root else None, recvs[r], root=root, count=count, dtype=dtype)
    torch.cuda.synchronize()
    for x in recvs:
        assert_bitwise(x.cpu().numpy(), send)
    p = comms[0].plan(False, root, count)
    if count * 4 <= (256 << 10):  # R#27: small calls run on the one BFS tree
        assert len(p["trees"]) == 1
        assert tuple(p["trees"][0]["parent"]) == OP.plan_shallow(g, False, root)["trees"][0]["parent"]
        assert comms[0].stats()["last_trees"] == 1
    else:
        assert len(p["trees"]) == 6
        assert comms[0].stats()["last_trees"] == 6


@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("count", [1, 4099, 30000, 65536])
def test_small_calls_on_link_graphs_shallow_tree(B, dtype, count):
    """R#27: small AllReduce / Broadcast on link graphs (DGX-1V, a 6-GPU
    fragment) run on one minimum-depth tree; fp32/bf16 AllReduce is bit-exact
    against the oracle's OWN plan_shallow (its reduction order), Broadcast is
    the root's bytes."""
    g8 = OG.dgx1v()
    frag, _ = OG.induced(g8, [0, 1, 3, 4, 5, 7])
    for g in (g8, frag):
        m = g[0]
        comms = make_comms(B, m, graph=B.Graph.from_pairs(m, g[1]))
        sends = synth.inputs(41 + m, m, count, dtype)
        got = run_allreduce(B, comms, sends, dtype, "sum")
        want = OC.allreduce(OP.plan_shallow(g, True), sends, dtype, "sum")
        for x in got:
            assert_bitwise(x, want)
        assert comms[0].stats()["last_trees"] == 1
        root = m - 1
        dsend = to_dev(sends[root], dtype)
        recvs = [sentinel(count, dtype) for _ in range(m)]
        for r, c in enumerate(comms):
            c.broadcast(dsend if r == root else None, recvs[r], root=root, count=count, dtype=dtype)
        torch.cuda.synchronize()
        for x in recvs:
            assert_bitwise(to_host(x, dtype), sends[root])
        for c in comms:
            c.destroy()


@pytest.mark.parametrize("per_rank", [0, 1])
def test_small_calls_on_link_graphs_tree_ll(B, per_rank):
    """R#27 + LL: calls that fit one LL slot (ll_max_bytes / m) on the single
    shallow tree take the low-latency protocol (no chunks, no flags): bit-exact
    against the oracle's plan_shallow for f32 / bf16 / i32 AllReduce and every
    Broadcast root, in one launch and in per-rank launches, interleaved with
    tree-executor calls and in place."""
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), launch_per_rank=per_rank)
    for dtype, count in (("f32", 1001), ("bf16", 3), ("i32", 4096)):
        sends = synth.inputs(77, 8, count, dtype)
        got = run_allreduce(B, comms, sends, dtype, "sum", inplace=(dtype == "i32"))
        assert comms[0].stats()["last_chunks"] == 0, "expected the LL protocol"
        want = OC.allreduce(OP.plan_shallow(g, True), sends, dtype, "sum")
        for x in got:
            assert_bitwise(x, want)
    count = 2049
    for root in range(8):
        src = synth.rank_input(78, root, count, "f32")
        bufs = [to_dev(src, "f32") if r == root else sentinel(count, "f32") for r in range(8)]
        for r, c in enumerate(comms):
            c.broadcast(bufs[r], bufs[r], root=root)
        torch.cuda.synchronize()
        assert comms[0].stats()["last_chunks"] == 0
        for x in bufs:
            assert_bitwise(to_host(x, "f32"), src)
        # a tree-executor call in between (shared epochs, alternating LL parity)
        big = synth.inputs(79, 8, 70001, "i32")
        gb = run_allreduce(B, comms, big, "i32", "sum")
        assert comms[0].stats()["last_chunks"] > 0
        for x in gb:
            assert_bitwise(x, OC.naive_reduce(big, "i32", "sum"))
    for c in comms:
        c.destroy()


def test_config2_dgx1v_broadcast_bf16_inplace(B):
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]))
    count = 300001
    send = synth.rank_input(2, 5, count, "bf16")
    bufs = [to_dev(send, "bf16") if r == 5 else sentinel(count, "bf16") for r in range(8)]
    for r, c in enumerate(comms):
        c.broadcast(bufs[r], bufs[r], root=5)
    torch.cuda.synchronize()
    for x in bufs:
        assert_bitwise(to_host(x, "bf16"), send)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_dgx1v_allreduce_multilevel_tree_order(B, dtype):
    g = OG.dgx1v()
    G = B.Graph.from_pairs(8, g[1])
    comms = make_comms(B, 8, graph=G, chunk_bytes=16384)
    count = 200003
    sends = synth.inputs(21, 8, count, dtype)
    got = run_allreduce(B, comms, sends, dtype, "sum")
    plan = oracle_plan_from_json(comms[0].plan(True, 0, count, dtype))
    assert max(t["parent"].count(-1) for t in plan["trees"]) == 1
    want = OC.allreduce(plan, sends, dtype, "sum")
    for x in got:
        assert_bitwise(x, want)
    # tolerance vs the naive-order sum (north_star): |gpu - naive| <= rtol * sum|x|
    rtol = 1e-5 if dtype == "f32" else 1e-2
    w = OC.bf16_to_f32(want) if dtype == "bf16" else want
    naive = OC.naive_reduce(sends, dtype, "sum")
    nv = OC.bf16_to_f32(naive) if dtype == "bf16" else naive
    absum = sum(np.abs(OC.bf16_to_f32(s) if dtype == "bf16" else s).astype(np.float64) for s in sends)
    assert np.all(np.abs(w.astype(np.float64) - nv) <= rtol * absum + 1e-30)


# Multi-level AllReduce plans the library and the oracle's paper pipeline
# (MWU runs -> ILP ladder) choose identically (tests/test_capi_cpu.py
# checks the others against it): the GPU result is compared with the oracle's
# evaluation of its OWN plan.  DGX-1V's full 8-GPU AllReduce is not among them
# (both pick 9 trees of 27/8, different ones).
OWN_PLAN_GRAPHS = [("dgx1p", list(range(8))), ("dgx1p", [0, 1, 3, 4, 5, 7]),
                   ("dgx1v", [2, 3, 6, 7]), ("dgx1v", [1, 4, 5, 6])]


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("machine,ids", OWN_PLAN_GRAPHS)
def test_multilevel_allreduce_against_the_oracles_own_plan(B, machine, ids, dtype):
    full = OG.dgx1v() if machine == "dgx1v" else OG.dgx1p()
    g, _ = OG.induced(full, ids)
    m = len(ids)
    own = OP.plan_allreduce_graph(g)
    assert own["accepted"] and max(t["depth"] for t in own["trees"]) >= 2
    comms = make_comms(B, m, graph=B.Graph.from_pairs(m, g[1]), chunk_bytes=16384)
    count = 300007            # > shallow_max_bytes (R#27) in both dtypes: the packed plan
    lib = comms[0].plan(True, 0, count, dtype)
    assert [tuple(t["parent"]) for t in lib["trees"]] == [t["parent"] for t in own["trees"]]
    assert [tuple(t["weight"]) for t in lib["trees"]] == \
        [(t["weight"].numerator, t["weight"].denominator) for t in own["trees"]]
    sends = synth.inputs(23, m, count, dtype)
    got = run_allreduce(B, comms, sends, dtype, "sum")
    want = OC.allreduce(own, sends, dtype, "sum")
    for x in got:
        assert_bitwise(x, want)
    for c in comms:
        c.destroy()


def test_dgx1v_allreduce_int_exact_and_fragments(B):
    g = OG.dgx1v()
    # fragmented allocations (config 4 secondary): induced sub-graphs
    for nodes in ([0, 1, 4], [0, 1, 3, 4, 5, 7], [2, 3, 6, 7], [1, 4, 5, 6], list(range(8))):
        sub, _ = OG.induced(g, nodes)
        m = len(nodes)
        comms = make_comms(B, m, graph=B.Graph.from_pairs(m, sub[1]), chunk_bytes=8192)
        count = 50021
        sends = synth.inputs(4, m, count, "i32")
        got = run_allreduce(B, comms, sends, "i32", "sum")
        want = OC.naive_reduce(sends, "i32", "sum")
        for x in got:
            assert_bitwise(x, want)
        mx = run_allreduce(B, comms, synth.inputs(5, m, count, "f32"), "f32", "max")
        wmx = OC.naive_reduce(synth.inputs(5, m, count, "f32"), "f32", "max")
        for x in mx:
            assert_bitwise(x, wmx)
        for c in comms:
            c.destroy()


def test_switch_broadcast_both_variants(B):
    m = 8
    for count, dtype in ((1000, "f32"), (3 * (1 << 20) + 1, "bf16")):   # star / two-level trees
        comms = make_comms(B, m)
        for root in (0, 6):
            send = synth.rank_input(9, root, count, dtype)
            dsend = to_dev(send, dtype)
            recvs = [sentinel(count, dtype) for _ in range(m)]
            for r, c in enumerate(comms):
                c.broadcast(dsend if r == root else None, recvs[r], root=root, count=count, dtype=dtype)
            torch.cuda.synchronize()
            for x in recvs:
                assert_bitwise(to_host(x, dtype), send)


def test_back_to_back_calls_and_epochs(B):
    # many calls without host sync: flags are epoch-monotonic, never reset
    m, count = 8, 65537
    comms = make_comms(B, m, chunk_bytes=8192)
    sends = synth.inputs(80, m, count, "f32")
    dsend = [to_dev(s, "f32") for s in sends]
    outs = [[torch.empty_like(d) for d in dsend] for _ in range(6)]
    for k in range(6):
        for r, c in enumerate(comms):
            c.allreduce(dsend[r], outs[k][r], op="sum")
    torch.cuda.synchronize()
    want = OC.naive_reduce(sends, "f32", "sum")
    for k in range(6):
        for x in outs[k]:
            assert_bitwise(x.cpu().numpy(), want)


def test_errors(B):
    comms = make_comms(B, 2)
    x = torch.zeros(16, device="cuda")
    with pytest.raises(B.BlinkError) as e:
        comms[0].broadcast(x, x, root=7)
    assert e.value.code == 4
    comms[0].allreduce(x, x, op="sum")
    with pytest.raises(B.BlinkError) as e:          # rank 1 disagrees on count
        comms[1].allreduce(x[:8], x[:8], op="sum")
    assert e.value.code == 5


# ----------------------------------------------------------------- full size, bench launch config
def test_fullsize_config3_sampled(B):
    """BASELINE config 3 at the bench size: 8 ranks x 256 MiB fp32, the exact
    launch configuration bench.py times; 65536 sampled outputs checked against
    the oracle's naive-order (= one-hop tree-order) sum."""
    import bench
    m, count = 8, bench.DEFAULT_COUNT
    comms = make_comms(B, m)
    sends = [synth.device_input(3, r, count, "f32") for r in range(m)]
    recvs = [torch.empty_like(s) for s in sends]
    for r, c in enumerate(comms):
        c.allreduce(sends[r], recvs[r], op="sum")
    torch.cuda.synchronize()
    idx = torch.from_numpy(np.random.default_rng(0).integers(0, count, 65536)).cuda()
    cols = [s[idx].cpu().numpy() for s in sends]
    want = OC.naive_reduce(cols, "f32", "sum")
    for r in range(m):
        assert_bitwise(recvs[r][idx].cpu().numpy(), want)
    # the last element and a tail window
    tail = [s[-37:].cpu().numpy() for s in sends]
    assert_bitwise(recvs[0][-37:].cpu().numpy(), OC.naive_reduce(tail, "f32", "sum"))


def test_cuda_graph_capture_and_replay(B):
    """Epochs live in device memory, so a captured call replays correctly
    (warm-up call first: the first call of a size uploads its tables)."""
    m, count = 8, 100003
    comms = make_comms(B, m)
    dsend = [torch.empty(count, device="cuda") for _ in range(m)]
    drecv = [torch.empty(count, device="cuda") for _ in range(m)]
    for r, c in enumerate(comms):          # warm-up (eager)
        c.allreduce(dsend[r], drecv[r])
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for r, c in enumerate(comms):
            c.allreduce(dsend[r], drecv[r])
    for it in range(4):
        sends = synth.inputs(90 + it, m, count, "f32")
        for d, s in zip(dsend, sends):
            d.copy_(torch.from_numpy(s))
        g.replay()
        torch.cuda.synchronize()
        want = OC.naive_reduce(sends, "f32", "sum")
        for x in drecv:
            assert_bitwise(x.cpu().numpy(), want)
    # eager calls after replays still agree on epochs
    for r, c in enumerate(comms):
        c.allreduce(dsend[r], drecv[r], op="max")
    torch.cuda.synchronize()
    want = OC.naive_reduce(sends, "f32", "max")
    for x in drecv:
        assert_bitwise(x.cpu().numpy(), want)


# ----------------------------------------------------------------- NEXT-3: ReduceScatter / AllGather
@pytest.mark.parametrize("m", [2, 3, 8])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
@pytest.mark.parametrize("B_", [1, 5, 4096, 33333])      # 16-byte aligned blocks and ragged ones
def test_reduce_scatter_and_allgather(B, m, dtype, B_):
    comms = make_comms(B, m, chunk_bytes=8192)
    sends = synth.inputs(100 + m, m, m * B_, dtype)
    ds = [to_dev(s, dtype) for s in sends]
    rs = [sentinel(B_, dtype) for _ in range(m)]
    for r, c in enumerate(comms):
        c.reduce_scatter(ds[r], rs[r], op="sum", recvcount=B_, dtype=dtype)
    torch.cuda.synchronize()
    want = OC.reduce_scatter(sends, dtype, "sum")
    for r in range(m):
        assert_bitwise(to_host(rs[r], dtype), want[r])
    # AllGather of the reduced blocks reproduces the one-hop AllReduce
    ag = [sentinel(m * B_, dtype) for _ in range(m)]
    for r, c in enumerate(comms):
        c.allgather(rs[r], ag[r], sendcount=B_, dtype=dtype)
    torch.cuda.synchronize()
    full = OC.allgather(want)
    assert_bitwise(full, OC.naive_reduce(sends, dtype, "sum"))
    for r in range(m):
        assert_bitwise(to_host(ag[r], dtype), full)


def test_allgather_inplace_and_rs_max(B):
    m, B_ = 5, 12345
    comms = make_comms(B, m)
    sends = synth.inputs(110, m, B_, "f32")
    bufs = [sentinel(m * B_, "f32") for _ in range(m)]
    for r in range(m):
        bufs[r][r * B_:(r + 1) * B_] = torch.from_numpy(sends[r]).cuda()
    for r, c in enumerate(comms):
        c.allgather(bufs[r][r * B_:(r + 1) * B_], bufs[r], sendcount=B_)
    torch.cuda.synchronize()
    for x in bufs:
        assert_bitwise(x.cpu().numpy(), OC.allgather(sends))
    big = synth.inputs(111, m, m * B_, "f32")
    ds = [to_dev(s, "f32") for s in big]
    out = [sentinel(B_, "f32") for _ in range(m)]
    for r, c in enumerate(comms):
        c.reduce_scatter(ds[r], out[r], op="max")
    torch.cuda.synchronize()
    want = OC.reduce_scatter(big, "f32", "max")
    for r in range(m):
        assert_bitwise(out[r].cpu().numpy(), want[r])


def test_block_collectives_on_multiserver_graphs_are_unsupported(B):
    g = OG.dgx1v()
    servers = [[0, 1, 2, 3], [4, 5, 6, 7]]
    comms = make_comms(B, 8, graph=B.Graph.multi_server(8, g[1], servers))
    x = torch.zeros(8 * 16, device="cuda")
    y = torch.zeros(16, device="cuda")
    for r, c in enumerate(comms):
        if r < 7:
            c.reduce_scatter(x, y)
        else:
            with pytest.raises(B.BlinkError) as e:
                c.reduce_scatter(x, y)
            assert e.value.code == 9


def test_miad_autotune_changes_chunking_not_results(B):
    """NEXT-2: with cfg.autotune the chunk size moves across calls (MIAD,
    P:526-535) while every call stays bit-exact (chunking never changes the
    per-element operations)."""
    m, count = 8, (2 << 20) + 7
    comms = make_comms(B, m, autotune=1)
    sends = synth.inputs(120, m, count, "f32")
    want = OC.naive_reduce(sends, "f32", "sum")
    ds = [to_dev(s, "f32") for s in sends]
    out = [torch.empty_like(d) for d in ds]
    chunks = set()
    for it in range(14):
        for r, c in enumerate(comms):
            c.allreduce(ds[r], out[r])
        torch.cuda.synchronize()
        chunks.add(comms[0].stats()["last_chunks"])
        if it % 4 == 0 or it == 13:
            for x in out:
                assert_bitwise(x.cpu().numpy(), want)
    assert len(chunks) >= 2          # the tuner explored several chunk sizes


# ----------------------------------------------------------------- NEXT-4: three-phase multi-server
@pytest.mark.parametrize("servers", [[[0, 1, 3], [2, 4, 5, 6, 7]], [[0, 1, 2, 3], [4, 5, 6, 7]]])
def test_multiserver_three_phase_allreduce(B, servers):
    """2 emulated servers (the paper's 3+5 split, P:715-721, and 4+4) on one
    GPU: exact int32, and fp32 bit-exact vs the oracle's tree-order evaluation
    of the library's plan plus the naive-sum tolerance."""
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.multi_server(8, g[1], servers), chunk_bytes=16384)
    count = 300007
    isends = synth.inputs(130, 8, count, "i32")
    for x in run_allreduce(B, comms, isends, "i32", "sum"):
        assert_bitwise(x, OC.naive_reduce(isends, "i32", "sum"))
    sends = synth.inputs(131, 8, count, "f32")
    got = run_allreduce(B, comms, sends, "f32", "sum")
    plan = oracle_plan_from_json(comms[0].plan(True, 0, count, "f32"))
    want = OC.allreduce(plan, sends, "f32", "sum")
    for x in got:
        assert_bitwise(x, want)
    absum = sum(np.abs(s).astype(np.float64) for s in sends)
    assert np.all(np.abs(want.astype(np.float64) - OC.naive_reduce(sends, "f32", "sum")) <= 1e-5 * absum + 1e-30)


# ----------------------------------------------------------------- full sizes of the other configs
def _sample_check(sends, recvs, op, dtype, nsamp=32768, seed=0):
    count = sends[0].numel()
    idx = torch.from_numpy(np.random.default_rng(seed).integers(0, count, nsamp)).cuda()
    idx = torch.cat([idx, torch.arange(max(0, count - 19), count, device="cuda")])
    cols = [to_host(s[idx], dtype) for s in sends]
    want = OC.naive_reduce(cols, dtype, op)
    for r in recvs:
        assert_bitwise(to_host(r[idx], dtype), want)


def test_fullsize_config2_dgx1v_broadcast_1gib(B):
    """Config 2 at its top size: 1 GiB Broadcast over the 6 emulated DGX-1V
    trees; every byte compared (device-side equality with the root's input)."""
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), timeout_s=60.0)
    count = (1 << 30) // 4 + 3
    send = synth.device_input(2, 0, count, "f32")
    recvs = [torch.full_like(send, float("nan")) for _ in range(8)]
    for r, c in enumerate(comms):
        c.broadcast(send if r == 0 else None, recvs[r], root=0)
    torch.cuda.synchronize()
    for x in recvs:
        assert torch.equal(x.view(torch.int32), send.view(torch.int32))


def test_fullsize_config3_bf16_1gib_and_config4_m7(B):
    for m, dtype, nbytes in ((8, "bf16", 1 << 30), (7, "f32", 1 << 30)):
        comms = make_comms(B, m, timeout_s=60.0)
        count = nbytes // OC.ESIZE[dtype]
        sends = [synth.device_input(3, r, count, dtype) for r in range(m)]
        recvs = [torch.empty_like(s) for s in sends]
        for r, c in enumerate(comms):
            c.allreduce(sends[r], recvs[r])
        torch.cuda.synchronize()
        _sample_check(sends, recvs, "sum", dtype)
        del sends, recvs
        for c in comms:
            c.destroy()
        torch.cuda.empty_cache()


def test_fullsize_config5_vgg16_bucket_sequence(B):
    """Config 5: the VGG-16 DDP bucket sequence (App. C) back to back, in place,
    at m = 8; every bucket sampled against the oracle."""
    m = 8
    comms = make_comms(B, m, timeout_s=60.0)
    for dtype in ("f32", "bf16"):
        buckets = synth.BUCKETS[("vgg16", dtype)]
        ins = [[synth.device_input(50 + i, r, n, dtype) for r in range(m)] for i, n in enumerate(buckets)]
        outs = [[x.clone() for x in b] for b in ins]
        for b in outs:
            for r, c in enumerate(comms):
                c.allreduce(b[r])                 # in place, back to back
        torch.cuda.synchronize()
        for b_in, b_out in zip(ins, outs):
            _sample_check(b_in, b_out, "sum", dtype, nsamp=8192)
        del ins, outs
        torch.cuda.empty_cache()


def test_device_trace_api(B):
    """BLINK_TRACE: per-CTA %globaltimer stamps of the last launch, ordered."""
    import os
    os.environ["BLINK_TRACE"] = "1"
    try:
        m, count = 8, 1 << 20
        comms = make_comms(B, m)
        xs = [torch.randn(count, device="cuda") for _ in range(m)]
        for r, c in enumerate(comms):
            c.allreduce(xs[r])
        torch.cuda.synchronize()
        tr = comms[0].trace()
        assert len(tr) == comms[0].stats()["last_ctas"] > 0
        for t in tr:
            stamps = [x for x in (t[0], t[1], t[2], t[6], t[7]) if x]
            assert stamps == sorted(stamps) and t[0] > 0
    finally:
        del os.environ["BLINK_TRACE"]


@pytest.mark.parametrize("m", [2, 3, 8])
@pytest.mark.parametrize("B_", [1, 6, 4096, 25001])
def test_gather(B, m, B_):
    comms = make_comms(B, m, chunk_bytes=16384)
    for root in sorted({0, m - 1, m // 2}):
        sends = synth.inputs(140 + root, m, B_, "f32")
        ds = [to_dev(s, "f32") for s in sends]
        out = sentinel(m * B_, "f32")
        for r, c in enumerate(comms):
            c.gather(ds[r], out if r == root else None, root=root, sendcount=B_, dtype="f32")
        torch.cuda.synchronize()
        assert_bitwise(out.cpu().numpy(), OC.gather(sends, root)[root])


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_sixteen_ranks_max(B, dtype):
    """kMaxRanks = 16 (a DGX-2-sized switch): one-hop AllReduce with
    16 sources per root (2-stage ring of 4 KiB tiles)."""
    m, count = 16, 16 * 3000 + 5
    comms = make_comms(B, m)
    sends = synth.inputs(150, m, count, dtype)
    got = run_allreduce(B, comms, sends, dtype, "sum")
    want = OC.allreduce(OP.plan_switch_allreduce(m), sends, dtype, "sum")
    for g in got:
        assert_bitwise(g, want)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_avg_multilevel_ll_and_reduce_scatter(B, dtype):
    """R#28 AVG: bit-exact vs the oracle (sum along the tree, one division at
    the root before its rounding) on DGX-1V's multi-level trees (tree
    executor, misaligned LSU path), the shallow tree in the LL protocol, the
    one-hop LL protocol, and ReduceScatter."""
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]), chunk_bytes=16384)
    for count in (200003, 1001):
        sends = synth.inputs(91, 8, count, dtype)
        got = run_allreduce(B, comms, sends, dtype, "avg")
        plan = oracle_plan_from_json(comms[0].plan(True, 0, count, dtype))
        want = OC.allreduce(plan, sends, dtype, "avg")
        for x in got:
            assert_bitwise(x, want)
    # misaligned buffers take the LSU path (reduce_range / Scalar)
    count = 50001
    sends = synth.inputs(92, 8, count, dtype)
    es = OC.ESIZE[dtype]
    dsend = []
    for s_ in sends:
        raw = torch.zeros(count * es + 16, dtype=torch.uint8, device="cuda")
        v = raw[es:es + count * es].view(TORCH_DT[dtype])
        v.copy_(to_dev(s_, dtype))
        dsend.append(v)
    drecv = [sentinel(count, dtype, offset=es) for _ in range(8)]
    for r, c in enumerate(comms):
        c.allreduce(dsend[r], drecv[r], op="avg", count=count, dtype=dtype)
    torch.cuda.synchronize()
    want = OC.allreduce(oracle_plan_from_json(comms[0].plan(True, 0, count, dtype)), sends, dtype, "avg")
    for x in drecv:
        assert_bitwise(to_host(x, dtype), want)
    for c in comms:
        c.destroy()
    comms = make_comms(B, 8)
    for count in (1001, 70001):   # one-hop LL, then the merged tree executor
        sends = synth.inputs(93, 8, count, dtype)
        got = run_allreduce(B, comms, sends, dtype, "avg")
        want = OC.allreduce(OP.plan_switch_allreduce(8), sends, dtype, "avg")
        for x in got:
            assert_bitwise(x, want)
    Bk = 4099
    rs = synth.inputs(94, 8, 8 * Bk, dtype)
    full = [to_dev(x, dtype) for x in rs]
    outs = [sentinel(Bk, dtype) for _ in range(8)]
    for r, c in enumerate(comms):
        c.reduce_scatter(full[r], outs[r], op="avg")
    torch.cuda.synchronize()
    blocks = OC.reduce_scatter(rs, dtype, "avg")
    for r in range(8):
        assert_bitwise(to_host(outs[r], dtype), blocks[r])
    for c in comms:
        c.destroy()


# ----------------------------------------------------------------- NEXT-3 on link graphs
LINK_GRAPHS = [("dgx1v", list(range(8))), ("dgx1v", [0, 1, 3, 4, 5, 7]), ("dgx1p", [1, 4, 5, 6]),
               ("dgx1p", [0, 1, 4])]


@pytest.mark.parametrize("machine,ids", LINK_GRAPHS)
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_link_graph_allgather_and_gather(B, machine, ids, dtype):
    """AllGather ("AllReduce without a reduction function") and Gather ("the
    inverse of Broadcast") on packed link graphs: multi-level trees,
    relays forwarding other ranks' blocks (Gather relays with recv = NULL go
    through the library's scratch).  Exact against the oracle's definitions."""
    full = OG.dgx1v() if machine == "dgx1v" else OG.dgx1p()
    g, _ = OG.induced(full, ids)
    m = len(ids)
    comms = make_comms(B, m, graph=B.Graph.from_pairs(m, g[1]), chunk_bytes=8192)
    for B_ in (1, 4099, 65536):
        sends = synth.inputs(150 + B_ % 7, m, B_, dtype)
        ds = [to_dev(s, dtype) for s in sends]
        outs = [sentinel(m * B_, dtype) for _ in range(m)]
        for r, c in enumerate(comms):
            c.allgather(ds[r], outs[r], sendcount=B_, dtype=dtype)
        torch.cuda.synchronize()
        want = OC.allgather(sends)
        for o in outs:
            assert_bitwise(to_host(o, dtype), want)
        for root in sorted({0, m - 1}):
            out = sentinel(m * B_, dtype)
            for r, c in enumerate(comms):
                c.gather(ds[r], out if r == root else None, root=root, sendcount=B_, dtype=dtype)
            torch.cuda.synchronize()
            assert_bitwise(to_host(out, dtype), OC.gather(sends, root)[root])
    assert comms[0].stats()["last_trees"] == m
    # ReduceScatter (the reduce half, inner ranks relaying partials): int32 and
    # MIN/MAX exact; fp32/bf16 bit-exact against the oracle's tree-order
    # evaluation of each block's tree
    B_ = 20011
    rsends = synth.inputs(155, m, m * B_, dtype)
    dr = [to_dev(s, dtype) for s in rsends]
    for op in ("sum", "max"):
        outs = [sentinel(B_, dtype) for _ in range(m)]
        for r, c in enumerate(comms):
            c.reduce_scatter(dr[r], outs[r], op=op, recvcount=B_, dtype=dtype)
        torch.cuda.synchronize()
        if dtype == "i32" or op == "max":
            want = OC.reduce_scatter(rsends, dtype, op)
        else:
            pj = B.plan_json(m, 2, 0, B_, dtype, graph=B.Graph.from_pairs(m, g[1]))
            want = [OC.allreduce(dict(trees=[dict(parent=tuple(t["parent"]), root=t["root"], weight=1)]),
                                 [s[j * B_:(j + 1) * B_] for s in rsends], dtype, op)
                    for j, t in enumerate(pj["trees"])]
        for r in range(m):
            assert_bitwise(to_host(outs[r], dtype), want[r])
    for c in comms:
        c.destroy()


def test_link_graph_allgather_in_place_and_depth(B):
    g = OG.dgx1v()
    comms = make_comms(B, 8, graph=B.Graph.from_pairs(8, g[1]))
    B_ = (1 << 20) + 3
    sends = synth.inputs(160, 8, B_, "f32")
    bufs = []
    for r in range(8):
        b = sentinel(8 * B_, "f32")
        b[r * B_:(r + 1) * B_] = to_dev(sends[r], "f32")
        bufs.append(b)
    for r, c in enumerate(comms):
        c.allgather(bufs[r][r * B_:(r + 1) * B_], bufs[r], sendcount=B_, dtype="f32")
    torch.cuda.synchronize()
    want = OC.allgather(sends)
    for b in bufs:
        assert_bitwise(to_host(b, "f32"), want)
    p = B.plan_json(8, 3, 0, B_, "f32", graph=B.Graph.from_pairs(8, g[1]))
    assert max(t["depth"] for t in p["trees"]) == 2          # DGX-1V: every rank within 2 hops
    for c in comms:
        c.destroy()
