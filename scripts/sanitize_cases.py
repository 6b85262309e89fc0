#!/usr/bin/env python
"""Small collectives for compute-sanitizer (memcheck / synccheck / racecheck):
one-hop AllReduce (TMA and LSU paths), emulated DGX-1V Broadcast and
multi-level AllReduce, ReduceScatter / AllGather, misaligned buffers, the LL
protocol (batched and per-rank launches) and a per-rank tree AllReduce.
Every result is checked against the oracle so a clean sanitizer run is also a
correct run."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
import synth  # noqa: E402
from oracle import collectives as OC  # noqa: E402
from oracle import graphs as OG  # noqa: E402


def check(got, want, what):
    g = got.cpu().numpy().view(np.uint32)
    if not np.array_equal(g, np.asarray(want).view(np.uint32)):
        raise SystemExit(f"MISMATCH {what}")


def main():
    cfg = B.config(timeout_s=120.0, chunk_bytes=8192)
    # one-hop AllReduce, aligned (TMA pipeline) and misaligned (LSU)
    m, n = 4, 20000 + 3
    comms = B.init_all([0] * m, cfg=cfg)
    sends = synth.inputs(200, m, n, "f32")
    xs = [torch.from_numpy(s).cuda() for s in sends]
    ys = [torch.empty_like(x) for x in xs]
    for r, c in enumerate(comms):
        c.allreduce(xs[r], ys[r])
    torch.cuda.synchronize()
    want = OC.naive_reduce(sends, "f32", "sum")
    for y in ys:
        check(y, want, "onehop")
    xm = []
    for s in sends:
        b = torch.empty(n + 1, device="cuda")
        b[1:] = torch.from_numpy(s).cuda()
        xm.append(b[1:])
    for r, c in enumerate(comms):
        c.allreduce(xm[r], ys[r])
    torch.cuda.synchronize()
    for y in ys:
        check(y, want, "misaligned")
    # RS / AG
    rs = [torch.empty(n, device="cuda") for _ in range(m)]
    big = synth.inputs(201, m, m * n, "f32")
    bx = [torch.from_numpy(s).cuda() for s in big]
    for r, c in enumerate(comms):
        c.reduce_scatter(bx[r], rs[r])
    ag = [torch.empty(m * n, device="cuda") for _ in range(m)]
    for r, c in enumerate(comms):
        c.allgather(rs[r], ag[r])
    torch.cuda.synchronize()
    for y in ag:
        check(y, OC.naive_reduce(big, "f32", "sum"), "rs+ag")
    for c in comms:
        c.destroy()
    # emulated DGX-1V Broadcast + multi-level AllReduce (int: exact under any tree)
    g = OG.dgx1v()
    # packed trees at this size (R#27's single shallow tree is checked below)
    packed = B.config(timeout_s=120.0, chunk_bytes=8192, shallow_max_bytes=0)
    comms = B.init_all([0] * 8, graph=B.Graph.from_pairs(8, g[1]), cfg=packed)
    src = synth.rank_input(202, 3, n, "f32")
    out = [torch.empty(n, device="cuda") for _ in range(8)]
    dsrc = torch.from_numpy(src).cuda()
    for r, c in enumerate(comms):
        c.broadcast(dsrc if r == 3 else None, out[r], root=3)
    torch.cuda.synchronize()
    for y in out:
        check(y, src, "dgx1v broadcast")
    isends = synth.inputs(203, 8, n, "i32")
    ix = [torch.from_numpy(s).cuda() for s in isends]
    iy = [torch.empty_like(x) for x in ix]
    for r, c in enumerate(comms):
        c.allreduce(ix[r], iy[r])
    torch.cuda.synchronize()
    for y in iy:
        check(y, OC.naive_reduce(isends, "i32", "sum"), "dgx1v allreduce")
    assert comms[0].stats()["last_trees"] > 1
    for c in comms:
        c.destroy()
    # small calls: the single minimum-depth tree (R#27), tree executor (64 KiB)
    # and tree LL protocol (16 KiB)
    comms = B.init_all([0] * 8, graph=B.Graph.from_pairs(8, g[1]), cfg=B.config(timeout_s=120.0))
    ns = 16001
    for r, c in enumerate(comms):
        c.allreduce(ix[r][:ns], iy[r][:ns])
    for r, c in enumerate(comms):
        c.broadcast(dsrc[:ns] if r == 3 else None, out[r][:ns], root=3)
    torch.cuda.synchronize()
    assert comms[0].stats()["last_chunks"] > 0
    for r in range(8):
        check(iy[r][:ns], OC.naive_reduce([s[:ns] for s in isends], "i32", "sum"), "dgx1v shallow allreduce")
        check(out[r][:ns], src[:ns], "dgx1v shallow broadcast")
    ns = 4099
    for r, c in enumerate(comms):
        c.allreduce(ix[r][:ns], iy[r][:ns])
    for r, c in enumerate(comms):
        c.broadcast(dsrc[:ns] if r == 3 else None, out[r][:ns], root=3)
    torch.cuda.synchronize()
    for r in range(8):
        check(iy[r][:ns], OC.naive_reduce([s[:ns] for s in isends], "i32", "sum"), "dgx1v shallow allreduce")
        check(out[r][:ns], src[:ns], "dgx1v shallow broadcast")
    assert comms[0].stats()["last_trees"] == 1
    for c in comms:
        c.destroy()
    # LL protocol (batched and per-rank launches) and the per-rank tree path
    for per_rank in (0, 1):
        comms = B.init_all([0] * 4, cfg=B.config(timeout_s=120.0, launch_per_rank=per_rank))
        for cnt in (1, 1001):
            ls = synth.inputs(204, 4, cnt, "f32")
            lx = [torch.from_numpy(s).cuda() for s in ls]
            ly = [torch.empty_like(x) for x in lx]
            for r, c in enumerate(comms):
                c.allreduce(lx[r], ly[r])
            for r, c in enumerate(comms):
                c.broadcast(lx[r] if r == 2 else None, lx[r], root=2)
            torch.cuda.synchronize()
            for r in range(4):
                check(ly[r], OC.naive_reduce(ls, "f32", "sum"), f"LL allreduce pr={per_rank}")
                check(lx[r], ls[2], f"LL broadcast pr={per_rank}")
        if per_rank:
            for r, c in enumerate(comms):
                c.allreduce(xs[r], ys[r])
            torch.cuda.synchronize()
            for y in ys:
                check(y, want, "per-rank tree allreduce")
        for c in comms:
            c.destroy()
    print("sanitize cases ok")


if __name__ == "__main__":
    main()
