#!/usr/bin/env python
"""Multi-process size sweep: Blink (one rank per process) next to NCCL.

    torchrun --nproc-per-node N --master-addr 127.0.0.1 scripts/sweep_mp.py [--out F] [--max-mib M]

Per size S (1 KiB .. M MiB, x4 steps) and collective (AllReduce SUM fp32,
Broadcast from rank 0): registered symmetric buffers, W warm-up calls, then
the mean of K calls on the launching stream (CUDA events), max over ranks.
NCCL (`torch.distributed` nccl group, same buffers, same stream) runs only
when the ranks sit on distinct GPUs; with BENCH_SAME_GPU=1 (every rank on
cuda:0, the 1-GPU box) the NCCL column is null -- NCCL refuses two ranks on
one device.  Rank 0 prints one JSON object (and writes --out).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1910_04940_b200 as B  # noqa: E402


def timed(fn, stream, warm, reps):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-mib", type=int, default=256)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    same = os.environ.get("BENCH_SAME_GPU") == "1"
    dev = 0 if same else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    nccl = None
    if not same:
        try:
            nccl = dist.new_group(backend="nccl")
        except Exception as e:  # pragma: no cover - depends on the box
            print(f"rank {rank}: no NCCL group: {e}", file=sys.stderr)
    ex = B.torch_exchange()
    comm = B.init_multiprocess(world, rank, dev, ex, cfg=B.config(timeout_s=60.0))
    maxb = args.max_mib << 20
    send = torch.randn(maxb // 4, device="cuda")
    recv = torch.empty_like(send)
    comm.register(send, maxb, ex)
    comm.register(recv, maxb, ex)
    stream = torch.cuda.current_stream()
    rows = []
    S = 1024
    while S <= maxb:
        cnt = S // 4
        reps = 200 if S <= (1 << 20) else (50 if S <= (64 << 20) else 10)
        x, y = send[:cnt], recv[:cnt]
        for coll in ("allreduce", "broadcast"):
            if coll == "allreduce":
                ours = lambda: comm.allreduce(x, y, op="sum", stream=stream)  # noqa: E731
                theirs = lambda: dist.all_reduce(y, group=nccl)  # noqa: E731
                busf = 2 * (world - 1) / world
            else:
                ours = lambda: comm.broadcast(x, y, root=0, stream=stream)  # noqa: E731
                theirs = lambda: dist.broadcast(y, src=0, group=nccl)  # noqa: E731
                busf = 1.0
            ms = timed(ours, stream, 5, reps)
            row = {"coll": coll, "bytes": S, "ms": round(ms, 5), "algbw": round(S / ms / 1e6, 2),
                   "busbw": round(S / ms / 1e6 * busf, 2)}
            if nccl is not None:
                if coll == "allreduce":
                    y.copy_(x)
                nms = timed(theirs, stream, 5, reps)
                row.update(nccl_ms=round(nms, 5), nccl_algbw=round(S / nms / 1e6, 2),
                           ratio=round(nms / ms, 3))
            rows.append(row)
        S *= 4
    comm.destroy()
    if rank == 0:
        out = {"world": world, "same_gpu": same, "device": torch.cuda.get_device_name(dev),
               "note": "mean of K calls (CUDA events, launching stream), max over ranks; "
                       "registered buffers; ratio = nccl_ms / blink_ms (>1: Blink faster)",
               "rows": rows}
        s = json.dumps(out)
        print(s)
        if args.out:
            with open(args.out, "w") as f:
                f.write(s + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
