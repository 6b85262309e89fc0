"""Worker for the multi-process tests (launched by torch.distributed.run).

MODE=cpu : host logic only (gloo): blob exchange, plan agreement, max-over-ranks.
MODE=gpu : the real multi-process path on GPU(s): CUDA-IPC flag/staging
           mappings, symmetric registration, entry handshake and exit waits.
           With BLINK_SAME_GPU=1 every rank uses cuda:0 (two processes
           time-share one B200; IPC maps the peer's allocations).
Exits non-zero on any mismatch against the oracle.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from oracle import collectives as OC  # noqa: E402
from oracle import graphs as OG  # noqa: E402
from oracle import packing as OP  # noqa: E402


def cpu_mode(rank, world):
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    ex = BD.exchange()
    blobs = ex(bytes([rank]) * 7)
    assert blobs == [bytes([r]) * 7 for r in range(world)], blobs
    d = BD.check_same_plan(world, True, 0, 12345, "bf16")
    tri, _ = OG.induced(OG.dgx1p(), [0, 1, 3])
    if world == 3:
        BD.check_same_plan(3, False, 0, 262144, graph=B.Graph.from_pairs(3, tri[1]))
    # a rank that would plan a different split must be detected on every rank
    try:
        BD.check_same_plan(world, True, 0, 1000 + 16 * rank)
        mismatch = False
    except B.BlinkError:
        mismatch = True
    assert mismatch
    assert BD.max_over_ranks(float(rank)) == world - 1
    print(f"rank {rank}: cpu ok {d[:12]}")


def to_dev(arr, dtype):
    a = np.ascontiguousarray(arr)
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
    return torch.from_numpy(a.copy()).cuda()


def gpu_mode(rank, world):
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    dev = 0 if os.environ.get("BLINK_SAME_GPU") == "1" else rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    comm = BD.init(cfg=B.config(timeout_s=60.0, staging_bytes=1 << 20), device=dev)
    ex = BD.exchange()

    def check(got, want, what):
        g = got.view(torch.int16).cpu().numpy().view(np.uint16) if got.dtype == torch.bfloat16 \
            else got.cpu().numpy()
        gb = g.view(np.uint16 if g.dtype.itemsize == 2 else np.uint32)
        wb = np.asarray(want).view(gb.dtype)
        bad = np.nonzero(gb != wb)[0]
        if bad.size:
            raise SystemExit(f"rank {rank}: {what}: {bad.size} mismatches, first {bad[:4]}")

    # 1) unregistered buffers -> staging path, several pieces (count > staging)
    count = 300001
    sends = synth.inputs(40, world, count, "f32")
    x = torch.from_numpy(sends[rank]).cuda()
    y = torch.full_like(x, float("nan"))
    comm.allreduce(x, y, op="sum")
    torch.cuda.synchronize()
    check(y, OC.naive_reduce(sends, "f32", "sum"), "staging allreduce f32")

    # 2) registered symmetric buffers (zero-copy), bf16, in place and out of place
    count = 1 << 20
    bs = synth.inputs(41, world, count, "bf16")
    xb = torch.from_numpy(bs[rank].view(np.int16).copy()).cuda().view(torch.bfloat16)
    yb = torch.empty_like(xb)
    comm.register(xb, xb.numel() * 2, ex)
    comm.register(yb, yb.numel() * 2, ex)
    comm.allreduce(xb, yb, op="sum")
    torch.cuda.synchronize()
    check(yb, OC.naive_reduce(bs, "bf16", "sum"), "registered allreduce bf16")
    comm.allreduce(xb, xb, op="max")
    torch.cuda.synchronize()
    check(xb, OC.naive_reduce(bs, "bf16", "max"), "registered in-place max bf16")

    # 3) broadcast from the last rank: registered recv, then staging
    root = world - 1
    src = synth.rank_input(42, root, count, "i32")
    xs = torch.from_numpy(src).cuda() if rank == root else None
    yr = torch.zeros(count, dtype=torch.int32, device="cuda")
    comm.register(yr, count * 4, ex)
    comm.broadcast(xs, yr, root=root, count=count, dtype="i32")
    torch.cuda.synchronize()
    check(yr, src, "registered broadcast")
    yu = torch.zeros(count + 5, dtype=torch.int32, device="cuda")
    comm.broadcast(xs, yu[:count], root=root, count=count, dtype="i32")
    torch.cuda.synchronize()
    check(yu[:count], src, "staging broadcast")

    # 4) many back-to-back calls (epochs) on registered buffers
    for _ in range(5):
        comm.allreduce(xb, yb, op="sum")
    torch.cuda.synchronize()
    check(yb, OC.naive_reduce([OC.naive_reduce(bs, "bf16", "max")] * world, "bf16", "sum"),
          "back-to-back")
    # 5) ReduceScatter / AllGather: staged (unregistered) then registered
    B_ = 70001
    rsends = synth.inputs(43, world, world * B_, "f32")
    xs_ = torch.from_numpy(rsends[rank]).cuda()
    out = torch.full((B_,), float("nan"), device="cuda")
    comm.reduce_scatter(xs_, out, op="sum")
    torch.cuda.synchronize()
    blocks = OC.reduce_scatter(rsends, "f32", "sum")
    check(out, blocks[rank], "staged reduce_scatter")
    ag = torch.full((world * B_,), float("nan"), device="cuda")
    comm.allgather(out, ag)
    torch.cuda.synchronize()
    check(ag, OC.allgather(blocks), "staged allgather")
    comm.register(xs_, xs_.numel() * 4, ex)
    comm.register(ag, ag.numel() * 4, ex)
    out2 = torch.full((B_,), float("nan"), device="cuda")
    comm.reduce_scatter(xs_, out2, op="max")
    comm.allgather(out2, ag)
    torch.cuda.synchronize()
    check(ag, OC.allgather(OC.reduce_scatter(rsends, "f32", "max")), "registered rs+ag")
    # 6) Gather to the last rank (staged: only the root holds a recv)
    gsends = synth.inputs(44, world, 9001, "f32")
    gx = torch.from_numpy(gsends[rank]).cuda()
    groot = world - 1
    gout = torch.full((world * 9001,), float("nan"), device="cuda") if rank == groot else None
    comm.gather(gx, gout, root=groot)
    torch.cuda.synchronize()
    if rank == groot:
        check(gout, OC.gather(gsends, groot)[groot], "staged gather")
    # 6b) Gather whose root recv IS registered while the other ranks pass
    # NULL: every rank must still take the same (staged) path
    greg = torch.full((world * 9001,), float("nan"), device="cuda")
    comm.register(greg, greg.numel() * 4, ex)          # collective: same size on every rank
    comm.gather(gx, greg if rank == groot else None, root=groot)
    torch.cuda.synchronize()
    if rank == groot:
        check(greg, OC.gather(gsends, groot)[groot], "gather into a registered root recv")
    # 7) low-latency protocol (small calls, unregistered buffers, no handshake):
    # AllReduce f32/bf16 (ragged), in place, Broadcast; then LL and tree calls
    # interleaved back to back (the epochs they share stay in step)
    for cnt, dt in ((1, "f32"), (1001, "f32"), (4099, "bf16")):
        ls = synth.inputs(45, world, cnt, dt)
        lx = to_dev(ls[rank], dt)
        ly = torch.empty_like(lx)
        la = torch.empty_like(lx)
        comm.allreduce(lx, la, op="avg")
        comm.allreduce(lx, ly, op="sum")
        comm.allreduce(lx, lx, op="max")
        torch.cuda.synchronize()
        check(la, OC.naive_reduce(ls, dt, "avg"), f"LL allreduce avg {dt} {cnt}")
        check(ly, OC.naive_reduce(ls, dt, "sum"), f"LL allreduce {dt} {cnt}")
        check(lx, OC.naive_reduce(ls, dt, "max"), f"LL in-place max {dt} {cnt}")
    bsrc = synth.rank_input(46, 0, 3333, "f32")
    bx = torch.from_numpy(bsrc).cuda() if rank == 0 else torch.zeros(3333, device="cuda")
    comm.broadcast(bx, bx, root=0)
    torch.cuda.synchronize()
    check(bx, bsrc, "LL broadcast")
    small = synth.inputs(47, world, 777, "f32")
    sx = torch.from_numpy(small[rank]).cuda()
    outs = []
    for k in range(6):
        o = torch.empty_like(sx)
        comm.allreduce(sx, o, op="sum")
        outs.append(o)
        comm.allreduce(xb, yb, op="sum")   # tree path (registered, 2 MiB)
    torch.cuda.synchronize()
    for o in outs:
        check(o, OC.naive_reduce(small, "f32", "sum"), "LL/tree interleaved")
    st = comm.stats()
    comm.destroy()
    print(f"rank {rank}: gpu ok launches={st['launches']} ctas={st['last_ctas']}")


def chain_mode(rank, world):
    """3 processes on the link graph 0 - 1 - 2 (R#27 shallow tree rooted at
    the centre, rank 1): small calls take the tree LL protocol across
    processes; five Broadcasts back to back from rank 0 (the root may run
    ahead of the leaves: the entry guard must hold it back); a packed-plan
    call in between."""
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    dev = 0 if os.environ.get("BLINK_SAME_GPU") == "1" else rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    G = B.Graph(3, [(0, 1, 1.0, 1), (1, 2, 1.0, 1)])
    comm = BD.init(graph=G, cfg=B.config(timeout_s=60.0, staging_bytes=1 << 20), device=dev)

    def check(got, want, what):
        gb = got.cpu().numpy().view(np.uint32)
        bad = np.nonzero(gb != np.asarray(want).view(np.uint32))[0]
        if bad.size:
            raise SystemExit(f"rank {rank}: {what}: {bad.size} mismatches, first {bad[:4]}")

    tree = OP.plan_shallow((3, {(0, 1): 1, (1, 0): 1, (1, 2): 1, (2, 1): 1}), True)
    assert tree["trees"][0]["root"] == 1
    for cnt in (1, 1001, 5003):
        ls = synth.inputs(48, world, cnt, "f32")
        lx = torch.from_numpy(ls[rank]).cuda()
        ly = torch.empty_like(lx)
        comm.allreduce(lx, ly, op="sum")
        torch.cuda.synchronize()
        assert comm.stats()["last_chunks"] == 0, "expected the LL protocol"
        check(ly, OC.allreduce(tree, ls, "f32", "sum"), f"tree LL allreduce {cnt}")
    srcs = [synth.rank_input(49 + k, 0, 2001, "f32") for k in range(5)]
    outs = [torch.from_numpy(srcs[k]).cuda() if rank == 0 else torch.zeros(2001, device="cuda")
            for k in range(5)]
    if rank != 0:
        torch.cuda._sleep(100_000_000)  # the leaves start late; the root must not overwrite
    for k in range(5):
        comm.broadcast(outs[k], outs[k], root=0)
    big = synth.inputs(50, world, 300001, "f32")
    bx = torch.from_numpy(big[rank]).cuda()
    by = torch.empty_like(bx)
    comm.allreduce(bx, by, op="sum")  # packed plan, tree executor
    torch.cuda.synchronize()
    for k in range(5):
        check(outs[k], srcs[k], f"tree LL broadcast {k}")
    # NEXT-3 on the chain: rank 1 relays; Gather to 0 (block 2 goes
    # 2 -> 1 -> 0 through the staging buffers) and AllGather
    gs = synth.inputs(52, world, 20001, "f32")
    gx = torch.from_numpy(gs[rank]).cuda()
    gout = torch.full((world * 20001,), float("nan"), device="cuda") if rank == 0 else None
    comm.gather(gx, gout, root=0)
    agout = torch.full((world * 20001,), float("nan"), device="cuda")
    comm.allgather(gx, agout)
    torch.cuda.synchronize()
    if rank == 0:
        check(gout, OC.gather(gs, 0)[0], "chain gather")
    check(agout, OC.allgather(gs), "chain allgather")
    # ReduceScatter on the chain: block 0's tree is 2 -> 1 -> 0 (rank 1 relays
    # partials through its staging relay area); int32 is exact in any order
    rsx = synth.inputs(55, world, world * 30001, "i32")
    rx = torch.from_numpy(rsx[rank]).cuda()
    ry = torch.zeros(30001, dtype=torch.int32, device="cuda")
    comm.reduce_scatter(rx, ry, op="sum")
    torch.cuda.synchronize()
    check(ry, OC.reduce_scatter(rsx, "i32", "sum")[rank], "chain reduce_scatter")
    comm.destroy()
    print(f"rank {rank}: chain ok")


def miad_mode(rank, world):
    """MIAD across processes (NEXT-2): rank 0 picks every
    autotuned call's chunk size and publishes it; every rank must chunk each
    call identically (same last_chunk_bytes), the size must change across
    calls, and every result stays bit-exact.  AllReduce and Broadcast calls
    interleave (one numbered sequence of autotuned calls across keys)."""
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    dev = 0 if os.environ.get("BLINK_SAME_GPU") == "1" else rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    comm = BD.init(cfg=B.config(timeout_s=60.0, autotune=1, staging_bytes=1 << 20), device=dev)
    ex = BD.exchange()
    count = 4 << 20
    sends = synth.inputs(51, world, count, "f32")
    x = torch.from_numpy(sends[rank]).cuda()
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    comm.register(x, count * 4, ex)
    comm.register(y, count * 4, ex)
    comm.register(z, count * 4, ex)
    want = OC.naive_reduce(sends, "f32", "sum")
    chunks, bchunks = [], []
    for k in range(14):
        y.fill_(float("nan"))
        comm.allreduce(x, y, op="sum")
        chunks.append(comm.stats()["last_chunk_bytes"])
        comm.broadcast(x if rank == 1 else None, z, root=1)
        bchunks.append(comm.stats()["last_chunk_bytes"])
        torch.cuda.synchronize()
        got = y.cpu().numpy()
        if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
            raise SystemExit(f"rank {rank}: MIAD call {k}: allreduce mismatch")
        if not np.array_equal(z.cpu().numpy().view(np.uint32), sends[1].view(np.uint32)):
            raise SystemExit(f"rank {rank}: MIAD call {k}: broadcast mismatch")
    allc = [None] * world
    dist.all_gather_object(allc, (chunks, bchunks))
    assert all(c == allc[0] for c in allc), allc
    assert len(set(chunks)) >= 2, chunks
    # a call captured into a CUDA graph neither times nor reads a slot: it
    # takes the last eager call's chunk on every rank; eager calls afterwards
    # continue the same numbered sequence
    torch.cuda.synchronize()
    dist.barrier()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.graph(g, stream=st):
        comm.allreduce(x, y, op="sum", stream=torch.cuda.current_stream())
    cap_chunk = comm.stats()["last_chunk_bytes"]
    for k in range(3):
        y.fill_(float("nan"))
        torch.cuda.synchronize()
        dist.barrier()
        g.replay()
        torch.cuda.synchronize()
        if not np.array_equal(y.cpu().numpy().view(np.uint32), want.view(np.uint32)):
            raise SystemExit(f"rank {rank}: MIAD captured replay {k}: allreduce mismatch")
    for k in range(2):
        y.fill_(float("nan"))
        comm.allreduce(x, y, op="sum")
        torch.cuda.synchronize()
        if not np.array_equal(y.cpu().numpy().view(np.uint32), want.view(np.uint32)):
            raise SystemExit(f"rank {rank}: MIAD eager call after capture {k}: allreduce mismatch")
    allcap = [None] * world
    dist.all_gather_object(allcap, cap_chunk)
    assert all(c == allcap[0] for c in allcap), allcap
    assert cap_chunk == chunks[-1], (cap_chunk, chunks[-1])
    del g
    comm.destroy()
    print(f"rank {rank}: miad ok {chunks} {bchunks} captured {cap_chunk}")


def nvls_mode(rank, world):
    """NEXT-1 across processes on distinct GPUs: rank 0's multicast object is
    joined by every rank at connect; AllReduce SUM within the north_star
    tolerance (f32) / exact (int32), Broadcast bitwise."""
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    comm = BD.init(cfg=B.config(timeout_s=60.0, nvls=1, nvls_bytes=4 << 20), device=dev)
    p = comm.plan(True, 0, 8 << 20, "f32")
    assert p["nvls"]["active"], p["nvls"]
    count = (3 << 20) + 7
    fs = synth.inputs(53, world, count, "f32")
    x = torch.from_numpy(fs[rank]).cuda()
    y = torch.empty_like(x)
    comm.allreduce(x, y, op="sum")
    ints = synth.inputs(54, world, count, "i32")
    xi = torch.from_numpy(ints[rank]).cuda()
    yi = torch.empty_like(xi)
    comm.allreduce(xi, yi, op="sum")
    z = torch.zeros_like(x)
    comm.broadcast(x if rank == 0 else None, z, root=0)
    torch.cuda.synchronize()
    naive = OC.naive_reduce(fs, "f32", "sum").astype(np.float64)
    absum = sum(np.abs(f.astype(np.float64)) for f in fs)
    if not np.all(np.abs(y.cpu().numpy().astype(np.float64) - naive) <= 1e-5 * absum + 1e-30):
        raise SystemExit(f"rank {rank}: NVLS f32 allreduce outside tolerance")
    if not np.array_equal(yi.cpu().numpy(), OC.naive_reduce(ints, "i32", "sum")):
        raise SystemExit(f"rank {rank}: NVLS i32 allreduce mismatch")
    if not np.array_equal(z.cpu().numpy().view(np.uint32), fs[0].view(np.uint32)):
        raise SystemExit(f"rank {rank}: NVLS broadcast mismatch")
    comm.destroy()
    print(f"rank {rank}: nvls ok")


def nvls_fallback_mode(rank, world):
    """cfg.nvls = 1 with every process on ONE GPU: a multicast team needs
    distinct devices, so the multi-process set-up (rank 0's object shared as
    a FABRIC handle or, without FABRIC support, a POSIX fd duplicated with
    pidfd_getfd) must end with NVLS off on EVERY rank, with the reason, and
    the collectives must run on the P2P stars, bit-exact."""
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    torch.cuda.set_device(0)
    comm = BD.init(cfg=B.config(timeout_s=60.0, nvls=1, nvls_bytes=4 << 20), device=0)
    p = comm.plan(True, 0, 1 << 20, "f32")
    assert p["nvls"]["active"] is False and p["nvls"]["note"].startswith("off"), p["nvls"]
    count = (1 << 18) + 3
    fs = synth.inputs(55, world, count, "f32")
    x = torch.from_numpy(fs[rank]).cuda()
    y = torch.empty_like(x)
    comm.allreduce(x, y, op="sum")
    torch.cuda.synchronize()
    want = OC.allreduce(OP.plan_switch_allreduce(world), fs, "f32", "sum")
    if not np.array_equal(y.cpu().numpy().view(np.uint32), want.view(np.uint32)):
        raise SystemExit(f"rank {rank}: allreduce after the NVLS fallback mismatch")
    comm.destroy()
    print(f"rank {rank}: nvls fallback ok ({p['nvls']['note']})")


def fuzz_mode(rank, world):
    """Randomized multi-process parity: every rank draws the same seeded
    sequence of graphs and collectives (switch or link graph, every
    collective, dtype and op, registered or staged buffers, LL and tree
    sizes, MIAD on or off) and checks each result against the oracle --
    the cross-process protocol (CUDA IPC, .sys flags, entry / exit waits,
    staging relays) on random configurations."""
    import random
    from fractions import Fraction
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    torch.cuda.set_device(0)
    ex = BD.exchange()
    base = int(os.environ.get("MP_FUZZ_BASE", "500"))
    n_cfg = int(os.environ.get("MP_FUZZ_N", "6"))
    done = 0
    for k in range(n_cfg):
        rng = random.Random(base + k)
        kind = rng.choice(["switch", "link"])
        graph = None
        pairs = None
        if kind == "link":
            while True:
                cap = {}
                for u in range(world):
                    for v in range(u + 1, world):
                        if rng.random() < 0.6:
                            cap[(u, v)] = cap[(v, u)] = rng.randint(1, 2)
                if OG.is_connected((world, cap)):
                    break
            graph = B.Graph.from_pairs(world, cap)
            pairs = cap
        comm = BD.init(graph=graph, cfg=B.config(timeout_s=60.0, staging_bytes=1 << 20,
                                                  autotune=int(rng.random() < 0.3)), device=0)
        for step in range(4):
            coll = rng.choice(["allreduce", "allreduce", "broadcast", "reduce_scatter", "allgather", "gather"])
            dtype = rng.choice(["f32", "bf16", "i32"])
            op = rng.choice(["sum", "max", "min"] + (["avg"] if coll == "allreduce" else []))
            count = rng.choice([1, 777, 65537, 300001, 1000003])  # 4 MB: TMA pipeline when registered
            reg = rng.random() < 0.4
            root = rng.randrange(world)
            n_in = world * count if coll == "reduce_scatter" else count
            sends = synth.inputs(base + 100 * k + step, world, n_in, dtype)
            x = to_dev(sends[rank], dtype)
            n_out = count if coll == "reduce_scatter" else (world * count if coll in ("allgather", "gather") else count)
            y = torch.zeros(n_out, dtype=x.dtype, device="cuda")
            if reg and coll != "gather":
                comm.register(x, x.numel() * x.element_size(), ex)
                comm.register(y, y.numel() * y.element_size(), ex)
            if coll == "allreduce":
                comm.allreduce(x, y, op=op, count=count, dtype=dtype)
            elif coll == "broadcast":
                comm.broadcast(x if rank == root else None, y, root=root, count=count, dtype=dtype)
            elif coll == "reduce_scatter":
                comm.reduce_scatter(x, y, op=op, recvcount=count, dtype=dtype)
            elif coll == "allgather":
                comm.allgather(x, y, sendcount=count, dtype=dtype)
            else:
                comm.gather(x, y if rank == root else None, root=root, sendcount=count, dtype=dtype)
            torch.cuda.synchronize()
            got = y.view(torch.int16).cpu().numpy().view(np.uint16) if dtype == "bf16" else y.cpu().numpy()
            what = f"cfg {k} step {step} {kind} {coll} {dtype} {op} n={count} reg={reg} root={root}"
            if coll == "broadcast":
                want = sends[root]
            elif coll in ("allgather", "gather"):
                if coll == "gather" and rank != root:
                    continue
                want = OC.allgather(sends)
            elif coll == "reduce_scatter":
                if kind == "switch" or dtype == "i32" or op in ("min", "max"):
                    want = OC.reduce_scatter(sends, dtype, op)[rank]
                else:
                    pj = B.plan_json(world, 2, 0, count, dtype, graph=graph)
                    t = pj["trees"][rank]
                    want = OC.allreduce(dict(trees=[dict(parent=tuple(t["parent"]), root=t["root"], weight=1)]),
                                        [sv[rank * count:(rank + 1) * count] for sv in sends], dtype, op)
            else:
                if dtype == "i32" or op in ("min", "max"):
                    want = OC.naive_reduce(sends, dtype, op)
                else:
                    p = comm.plan(True, 0, count, dtype)
                    want = OC.allreduce(dict(trees=[dict(parent=tuple(t["parent"]), root=t["root"],
                                                         weight=Fraction(*t["weight"])) for t in p["trees"]]),
                                        sends, dtype, op)
            gb = got.view(np.uint16 if got.dtype.itemsize == 2 else np.uint32)
            wb = np.asarray(want).view(gb.dtype)
            if not np.array_equal(gb, wb):
                bad = np.nonzero(gb != wb)[0]
                raise SystemExit(f"rank {rank}: {what}: {bad.size} mismatches, first {bad[:4]}")
            done += 1
        comm.destroy()
    print(f"rank {rank}: fuzz ok {done}")


def vmm_mode(rank, world):
    """Zero-copy registration of VMM memory (PyTorch expandable segments,
    PYTORCH_CUDA_ALLOC_CONF=expandable_segments:True set by the launcher):
    buffers straddling the allocator's physical chunks are exported chunk by
    chunk and mapped by the peers; a registered call is ONE launch (the staged
    path would take many with a 1 MiB staging buffer) and bit-exact."""
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    assert "expandable_segments:True" in os.environ.get("PYTORCH_CUDA_ALLOC_CONF", "")
    torch.cuda.set_device(0)
    comm = BD.init(cfg=B.config(timeout_s=60.0, staging_bytes=1 << 20, ll_max_bytes=0), device=0)
    ex = BD.exchange()
    pad = torch.empty(7 << 20, dtype=torch.uint8, device="cuda")  # push the next tensors across chunk edges
    count = (12 << 20) + 5                                       # 48 MiB of fp32: spans 3+ chunks
    fs = synth.inputs(56, world, count, "f32")
    x = torch.from_numpy(fs[rank]).cuda()
    y = torch.empty_like(x)
    comm.register(x, x.numel() * 4, ex)
    comm.register(y, y.numel() * 4, ex)
    l0 = comm.stats()["launches"]
    comm.allreduce(x, y, op="sum")
    torch.cuda.synchronize()
    assert comm.stats()["launches"] - l0 == 1, "expected the zero-copy path"
    if not np.array_equal(y.cpu().numpy().view(np.uint32), OC.naive_reduce(fs, "f32", "sum").view(np.uint32)):
        raise SystemExit(f"rank {rank}: VMM registered allreduce mismatch")
    comm.broadcast(x if rank == 1 else None, y, root=1)
    torch.cuda.synchronize()
    if not np.array_equal(y.cpu().numpy().view(np.uint32), fs[1].view(np.uint32)):
        raise SystemExit(f"rank {rank}: VMM registered broadcast mismatch")
    del pad
    comm.destroy()
    print(f"rank {rank}: vmm ok")


def fingerprint_mode(rank, world):
    """Ranks whose chunk tables differ (here BLINK_CHUNKS_PER_CTA on rank 1)
    would consume each other's flags for different byte ranges: blink_connect
    refuses the mix on every rank with BLINK_ERR_INVALID_USAGE."""
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    torch.cuda.set_device(0)
    if rank == 1:
        os.environ["BLINK_CHUNKS_PER_CTA"] = "7"
    try:
        BD.init(cfg=B.config(timeout_s=5.0), device=0)
        raise SystemExit(f"rank {rank}: connect accepted mismatched chunking")
    except B.BlinkError as e:
        assert e.code == 5 and "chunks differently" in str(e), e
    print(f"rank {rank}: fingerprint ok")


def timeout_mode(rank, world):
    """Failure detection: rank 1 never joins the collective; rank 0's flag
    waits time out (cfg.timeout_s), the launch aborts instead of hanging, and
    the next call on rank 0 reports BLINK_ERR_TIMEOUT."""
    import paper_1910_04940_b200 as B
    from paper_1910_04940_b200 import dist as BD
    torch.cuda.set_device(0)
    # the tree executor (entry-flag wait) and the LL protocol (data-line poll)
    for what, llmax in (("tree", 0), ("LL", 64 << 10)):
        comm = BD.init(cfg=B.config(timeout_s=1.0, ll_max_bytes=llmax), device=0)
        x = torch.ones(4096, device="cuda")
        if rank == 0:
            comm.allreduce(x)              # enqueued; the kernel waits for rank 1
            torch.cuda.synchronize()       # returns once the wait timed out
            try:
                comm.allreduce(x)
                raise SystemExit("rank 0: expected BLINK_ERR_TIMEOUT")
            except B.BlinkError as e:
                assert e.code == 10, e
            print(f"rank 0: {what} timeout ok")
        else:
            print(f"rank 1: skipped the {what} collective")
        dist.barrier()
        comm.destroy()
        dist.barrier()


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dist.init_process_group("gloo")
    try:
        mode = os.environ.get("MODE", "cpu")
        if mode == "cpu":
            cpu_mode(rank, world)
        elif mode == "timeout":
            timeout_mode(rank, world)
        elif mode == "chain":
            chain_mode(rank, world)
        elif mode == "fingerprint":
            fingerprint_mode(rank, world)
        elif mode == "miad":
            miad_mode(rank, world)
        elif mode == "nvls":
            nvls_mode(rank, world)
        elif mode == "nvls_fallback":
            nvls_fallback_mode(rank, world)
        elif mode == "fuzz":
            fuzz_mode(rank, world)
        elif mode == "vmm":
            vmm_mode(rank, world)
        else:
            gpu_mode(rank, world)
    finally:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
