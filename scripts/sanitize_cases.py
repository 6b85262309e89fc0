#!/usr/bin/env python
"""Small collectives for compute-sanitizer (memcheck / synccheck / racecheck).

One section per executor path, each with its thresholds pinned in its own
config so a later change of a default cannot silently move a case onto another
path (the round-1 script broke that way).  Every section checks which path ran
(`stats()`: LL calls report 0 chunks) and checks every result against the
oracle, so a clean sanitizer run is also a correct run.  It prints
"ok <section>" per section and "sanitize cases ok" at the end.

Sections: one-hop tree executor (TMA aligned, LSU misaligned), bf16, AVG,
ReduceScatter / AllGather, DGX-1V packed Broadcast and multi-level AllReduce,
the R#27 shallow tree on the tree executor, the shallow tree in the LL
protocol, NEXT-3 on the DGX-1V link graph (AllGather, Gather with relays,
ReduceScatter with relayed partials; batched and per-rank), switch LL (batched
and per-rank launches), per-rank tree AllReduce, work stealing across channels.
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
import synth  # noqa: E402
from oracle import collectives as OC  # noqa: E402
from oracle import graphs as OG  # noqa: E402
from oracle import packing as OP  # noqa: E402

T = 120.0  # flag-wait timeout: the sanitizers slow kernels down by 100x and more


def dev(a, dtype="f32"):
    a = np.ascontiguousarray(a)
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).cuda().view(torch.bfloat16)
    return torch.from_numpy(a.copy()).cuda()


def check(got, want, what):
    g = got.contiguous().view(torch.uint8).cpu().numpy().tobytes()
    if g != np.ascontiguousarray(want).tobytes():
        raise SystemExit(f"MISMATCH {what}")


def expect_path(comm, tree_executor, what):
    chunks = comm.stats()["last_chunks"]
    if tree_executor != (chunks > 0):
        raise SystemExit(f"WRONG PATH {what}: last_chunks={chunks}")


def allreduce(comms, xs, ys, op="sum"):
    for r, c in enumerate(comms):
        c.allreduce(xs[r], ys[r], op=op)
    torch.cuda.synchronize()


def onehop_sections():
    m, n = 4, 20000 + 3
    cfg = B.config(timeout_s=T, chunk_bytes=8192, ll_max_bytes=0)
    comms = B.init_all([0] * m, cfg=cfg)
    sends = synth.inputs(200, m, n, "f32")
    xs = [dev(s) for s in sends]
    ys = [torch.empty_like(x) for x in xs]
    allreduce(comms, xs, ys)
    want = OC.naive_reduce(sends, "f32", "sum")
    for y in ys:
        check(y, want, "onehop tma")
    expect_path(comms[0], True, "onehop tma")
    print("ok onehop TMA", flush=True)
    xm = []
    for s in sends:
        b = torch.empty(n + 1, device="cuda")
        b[1:] = torch.from_numpy(s).cuda()
        xm.append(b[1:])
    allreduce(comms, xm, ys)
    for y in ys:
        check(y, want, "onehop lsu")
    print("ok onehop LSU (misaligned)", flush=True)
    bs = synth.inputs(205, m, n, "bf16")
    bx = [dev(s, "bf16") for s in bs]
    by = [torch.empty_like(x) for x in bx]
    allreduce(comms, bx, by)
    for y in by:
        check(y, OC.allreduce(OP.plan_switch_allreduce(m), bs, "bf16", "sum"), "bf16")
    print("ok onehop bf16", flush=True)
    allreduce(comms, xs, ys, op="avg")
    for y in ys:
        check(y, OC.allreduce(OP.plan_switch_allreduce(m), sends, "f32", "avg"), "avg")
    print("ok onehop AVG", flush=True)
    rs = [torch.empty(n, device="cuda") for _ in range(m)]
    big = synth.inputs(201, m, m * n, "f32")
    bxs = [dev(s) for s in big]
    for r, c in enumerate(comms):
        c.reduce_scatter(bxs[r], rs[r])
    ag = [torch.empty(m * n, device="cuda") for _ in range(m)]
    for r, c in enumerate(comms):
        c.allgather(rs[r], ag[r])
    torch.cuda.synchronize()
    for y in ag:
        check(y, OC.naive_reduce(big, "f32", "sum"), "rs+ag")
    print("ok ReduceScatter + AllGather", flush=True)
    for c in comms:
        c.destroy()
    return sends, want


def dgx1v_sections(n=20000 + 3):
    g = OG.dgx1v()
    G = B.Graph.from_pairs(8, g[1])
    src = synth.rank_input(202, 3, n, "f32")
    dsrc = dev(src)
    out = [torch.empty(n, device="cuda") for _ in range(8)]
    isends = synth.inputs(203, 8, n, "i32")
    ix = [dev(s) for s in isends]
    iy = [torch.empty_like(x) for x in ix]
    # packed trees (R#27's single tree off), tree executor
    packed = B.config(timeout_s=T, chunk_bytes=8192, shallow_max_bytes=0, ll_max_bytes=0)
    comms = B.init_all([0] * 8, graph=G, cfg=packed)
    for r, c in enumerate(comms):
        c.broadcast(dsrc if r == 3 else None, out[r], root=3)
    torch.cuda.synchronize()
    for y in out:
        check(y, src, "dgx1v broadcast")
    expect_path(comms[0], True, "dgx1v broadcast")
    if comms[0].stats()["last_trees"] != 6:
        raise SystemExit("dgx1v broadcast: expected the 6 packed trees")
    allreduce(comms, ix, iy)
    for y in iy:
        check(y, OC.naive_reduce(isends, "i32", "sum"), "dgx1v allreduce")
    if comms[0].stats()["last_trees"] <= 1:
        raise SystemExit("dgx1v allreduce: expected packed trees")
    print("ok DGX-1V packed Broadcast + multi-level AllReduce", flush=True)
    for c in comms:
        c.destroy()
    # work stealing: 36 KiB chunks (TMA path, above the 32 KiB register-path
    # cap) give the 1-CTA channels > 3 rounds of chunks
    steal = B.config(timeout_s=T, chunk_bytes=36864, shallow_max_bytes=0, ll_max_bytes=0)
    comms = B.init_all([0] * 8, graph=G, cfg=steal)
    ns = 600000 + 3
    ssends = synth.inputs(204, 8, ns, "i32")
    sx = [dev(s) for s in ssends]
    sy = [torch.empty_like(x) for x in sx]
    allreduce(comms, sx, sy)
    for y in sy:
        check(y, OC.naive_reduce(ssends, "i32", "sum"), "dgx1v allreduce (stealing)")
    if comms[0].stats()["last_steal_channels"] <= 0:
        raise SystemExit("dgx1v allreduce: expected work stealing on")
    print("ok DGX-1V multi-level AllReduce with work stealing", flush=True)
    for c in comms:
        c.destroy()
    # R#27 shallow tree on the tree executor (LL off), 64 KiB
    shallow = B.config(timeout_s=T, shallow_max_bytes=256 << 10, ll_max_bytes=0)
    comms = B.init_all([0] * 8, graph=G, cfg=shallow)
    ns = 16001
    allreduce(comms, [x[:ns] for x in ix], [y[:ns] for y in iy])
    expect_path(comms[0], True, "shallow allreduce")
    for r, c in enumerate(comms):
        c.broadcast(dsrc[:ns] if r == 3 else None, out[r][:ns], root=3)
    torch.cuda.synchronize()
    expect_path(comms[0], True, "shallow broadcast")
    if comms[0].stats()["last_trees"] != 1:
        raise SystemExit("shallow: expected one tree")
    for r in range(8):
        check(iy[r][:ns], OC.naive_reduce([s[:ns] for s in isends], "i32", "sum"), "shallow allreduce")
        check(out[r][:ns], src[:ns], "shallow broadcast")
    print("ok DGX-1V shallow tree (tree executor)", flush=True)
    for c in comms:
        c.destroy()
    # the shallow tree in the LL protocol, 16 KiB
    lltree = B.config(timeout_s=T, shallow_max_bytes=256 << 10, ll_max_bytes=256 << 10)
    comms = B.init_all([0] * 8, graph=G, cfg=lltree)
    ns = 4099
    allreduce(comms, [x[:ns] for x in ix], [y[:ns] for y in iy])
    expect_path(comms[0], False, "LL tree allreduce")
    for r, c in enumerate(comms):
        c.broadcast(dsrc[:ns] if r == 3 else None, out[r][:ns], root=3)
    torch.cuda.synchronize()
    expect_path(comms[0], False, "LL tree broadcast")
    for r in range(8):
        check(iy[r][:ns], OC.naive_reduce([s[:ns] for s in isends], "i32", "sum"), "LL tree allreduce")
        check(out[r][:ns], src[:ns], "LL tree broadcast")
    print("ok DGX-1V shallow tree (LL protocol)", flush=True)
    for c in comms:
        c.destroy()


def link_block_sections():
    """NEXT-3 on the DGX-1V link graph: AllGather (multi-level trees), Gather
    (relays through scratch, recv = None off the root) and ReduceScatter
    (inner ranks relay partials, roots write recv, acks), batched and per-rank."""
    g = OG.dgx1v()
    G = B.Graph.from_pairs(8, g[1])
    n = 5003
    for per_rank in (0, 1):
        comms = B.init_all([0] * 8, graph=G, cfg=B.config(timeout_s=T, chunk_bytes=8192,
                                                          launch_per_rank=per_rank, ll_max_bytes=0))
        sends = synth.inputs(206, 8, n, "i32")
        xs = [dev(s) for s in sends]
        ag = [torch.zeros(8 * n, dtype=torch.int32, device="cuda") for _ in range(8)]
        for r, c in enumerate(comms):
            c.allgather(xs[r], ag[r])
        torch.cuda.synchronize()
        for y in ag:
            check(y, OC.allgather(sends), "link allgather")
        gout = torch.zeros(8 * n, dtype=torch.int32, device="cuda")
        for r, c in enumerate(comms):
            c.gather(xs[r], gout if r == 5 else None, root=5)
        torch.cuda.synchronize()
        check(gout, OC.gather(sends, 5)[5], "link gather")
        rsend = synth.inputs(207, 8, 8 * n, "i32")
        rx = [dev(s) for s in rsend]
        ry = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(8)]
        for r, c in enumerate(comms):
            c.reduce_scatter(rx[r], ry[r], op="sum")
        torch.cuda.synchronize()
        want = OC.reduce_scatter(rsend, "i32", "sum")
        for r in range(8):
            check(ry[r], want[r], "link reduce_scatter")
        expect_path(comms[0], True, "link reduce_scatter")
        print(f"ok DGX-1V AllGather / Gather / ReduceScatter ({'per-rank' if per_rank else 'batched'})",
              flush=True)
        for c in comms:
            c.destroy()


def ll_and_per_rank_sections(sends, want):
    for per_rank in (0, 1):
        comms = B.init_all([0] * 4, cfg=B.config(timeout_s=T, launch_per_rank=per_rank,
                                                 ll_max_bytes=256 << 10))
        for cnt in (1, 1001):
            ls = synth.inputs(204, 4, cnt, "f32")
            lx = [dev(s) for s in ls]
            ly = [torch.empty_like(x) for x in lx]
            allreduce(comms, lx, ly)
            # one launch holding every rank: AllReduce runs the merged register path
            expect_path(comms[0], per_rank == 0, f"LL allreduce pr={per_rank}")
            for r, c in enumerate(comms):
                c.broadcast(lx[r] if r == 2 else None, lx[r], root=2)
            torch.cuda.synchronize()
            expect_path(comms[0], False, f"LL broadcast pr={per_rank}")
            for r in range(4):
                check(ly[r], OC.naive_reduce(ls, "f32", "sum"), f"LL allreduce pr={per_rank}")
                check(lx[r], ls[2], f"LL broadcast pr={per_rank}")
        print(f"ok switch LL ({'per-rank' if per_rank else 'batched'} launches)", flush=True)
        for c in comms:
            c.destroy()
    # the multi-process protocol's tree executor: per-rank launches, LL off
    comms = B.init_all([0] * 4, cfg=B.config(timeout_s=T, launch_per_rank=1, ll_max_bytes=0,
                                             chunk_bytes=8192))
    xs = [dev(s) for s in sends]
    ys = [torch.empty_like(x) for x in xs]
    allreduce(comms, xs, ys)
    expect_path(comms[0], True, "per-rank tree allreduce")
    for y in ys:
        check(y, want, "per-rank tree allreduce")
    print("ok per-rank tree AllReduce", flush=True)
    for c in comms:
        c.destroy()


def main():
    sends, want = onehop_sections()
    dgx1v_sections()
    link_block_sections()
    ll_and_per_rank_sections(sends, want)
    print("sanitize cases ok", flush=True)


if __name__ == "__main__":
    main()
