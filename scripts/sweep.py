#!/usr/bin/env python
"""Size sweeps for every BASELINE.json config on one B200 (virtual ranks).

    python scripts/sweep.py [--out profiles/sweep_rNN.json] [--quick]

Rows: config, collective, plan, m, dtype, bytes per rank S, ms per call (CUDA
events, mean of `reps` back-to-back calls after warm-up), algBW = S/t,
busBW = algBW * f (f = 2(m-1)/m AllReduce, 1 Broadcast), and, because virtual
ranks share one HBM, the algorithmic HBM bytes per call and their fraction of
MEASURED_PEAKS.json hbm_gbs:
  AllReduce : 2 m S   (every send read once, every recv written once)
  Broadcast : (m+1) S (root send read once, every recv written once)
plus `plan_hbm_frac`: the HBM bytes the chosen plan must move (multi-hop
trees re-read partials / forwarded chunks) over the same time -- the
executor's efficiency on its plan.
Config 5 replays the App. C DDP bucket sequences back to back on one stream.
Times are device times of CUDA-graph replays (no host enqueue cost): `ms` per
call with up to 10 back-to-back calls per graph, `ms_one_call_per_graph` with
one (that adds a graph launch, ~8 us, to every call).
"""
import argparse
import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1910_04940_b200 as B  # noqa: E402
import synth  # noqa: E402
from oracle import graphs as OG  # noqa: E402  (topology presets only: the emulated link graphs)

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
TD = {"f32": torch.float32, "bf16": torch.bfloat16, "i32": torch.int32}
ES = {"f32": 4, "bf16": 2, "i32": 4}


def time_calls(fn, nbytes):
    """Device time per call of back-to-back calls: up to 10 calls are captured
    in one CUDA graph (epochs are device-resident, so replays are valid) and
    the graph is replayed; a graph launch has a fixed cost of its own
    (~8 us on this box), which one call per graph would measure instead of the
    collective (round 1's sweep did: every size up to 1 MiB read 8.3 us).
    Returns (ms per call in a 10-call graph, ms per call with one call per
    graph)."""
    per_graph = 10 if nbytes <= (64 << 20) else 2
    reps = 20 if nbytes <= (1 << 20) else (10 if nbytes <= (64 << 20) else 5)

    def measure(k, r):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(k):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(r):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (r * k)

    return measure(per_graph, reps), measure(1, reps)


def plan_traffic(plan, coll, esize):
    """HBM bytes the executor must move for this plan when every rank shares
    one HBM (virtual ranks): per tree of range S_i --
      AllReduce: REDUCE at v with k children reads (1+k) S_i and writes S_i
      (partial) or, at the root, (1+k) S_i (own + children's recv); an inner
      node's BCAST reads S_i and writes k S_i.
      Broadcast: the root reads S_i and writes (k+1) S_i (own recv + k
      children); an inner node reads S_i and writes k S_i."""
    tot = 0
    for t in plan["trees"]:
        Si = (t["hi"] - t["lo"]) * esize
        par = t["parent"]
        kids = {v: sum(1 for u in par if u == v) for v in range(len(par))}
        for v, k in kids.items():
            if k == 0:
                continue
            is_root = par[v] < 0
            if coll == "allreduce":
                tot += (1 + k) * Si + ((1 + k) * Si if is_root else Si)
                if not is_root:
                    tot += Si + k * Si
            else:
                tot += Si + (k + (1 if is_root else 0)) * Si
    return tot


def run_coll(comms, coll, S, dtype, root=0, tag=""):
    m = len(comms)
    cnt = max(1, S // ES[dtype])
    sends = [torch.randn(cnt, device="cuda").to(TD[dtype]) if dtype != "i32" else
             torch.randint(-1000, 1000, (cnt,), device="cuda", dtype=torch.int32) for _ in range(m)]
    recvs = [torch.empty_like(s) for s in sends]
    if coll == "allreduce":
        def fn():
            for r, c in enumerate(comms):
                c.allreduce(sends[r], recvs[r])
        hbm = 2 * m * cnt * ES[dtype]
        f = 2 * (m - 1) / m
    else:
        def fn():
            for r, c in enumerate(comms):
                c.broadcast(sends[root] if r == root else None, recvs[r], root=root)
        hbm = (m + 1) * cnt * ES[dtype]
        f = 1.0
    ms, ms1 = time_calls(fn, cnt * ES[dtype])
    Sb = cnt * ES[dtype]
    alg = Sb / (ms * 1e-3) / 1e9
    plan = comms[0].plan(coll == "allreduce", root, cnt, dtype)
    pt = plan_traffic(plan, coll, ES[dtype])
    return {"config": tag, "coll": coll, "m": m, "dtype": dtype, "bytes": Sb, "ms": round(ms, 5),
            "ms_one_call_per_graph": round(ms1, 5),
            "algbw": round(alg, 2), "busbw": round(alg * f, 2),
            "hbm_gbs": round(hbm / (ms * 1e-3) / 1e9, 1), "hbm_frac": round(hbm / (ms * 1e-3) / 1e9 / PEAK, 4),
            "plan_hbm_bytes": pt, "plan_hbm_frac": round(pt / (ms * 1e-3) / 1e9 / PEAK, 4),
            "trees": len(plan["trees"]), "ctas": plan["ctas"],
            "max_depth": max(t["depth"] for t in plan["trees"])}


def run_block(comms, coll, S, dtype, tag):
    """ReduceScatter / AllGather; S = full (m-block) buffer bytes per rank.
    Algorithmic HBM bytes: RS reads m*S, writes S; AG reads S, writes m*S."""
    m = len(comms)
    B = max(1, S // ES[dtype] // m)
    full = [torch.randn(m * B, device="cuda").to(TD[dtype]) for _ in range(m)]
    part = [torch.randn(B, device="cuda").to(TD[dtype]) for _ in range(m)]
    if coll == "reduce_scatter":
        def fn():
            for r, c in enumerate(comms):
                c.reduce_scatter(full[r], part[r])
    else:
        def fn():
            for r, c in enumerate(comms):
                c.allgather(part[r], full[r])
    Sb = m * B * ES[dtype]
    ms, ms1 = time_calls(fn, Sb)
    hbm = (m + 1) * Sb
    alg = Sb / (ms * 1e-3) / 1e9
    return {"config": tag, "coll": coll, "m": m, "dtype": dtype, "bytes": Sb, "ms": round(ms, 5),
            "ms_one_call_per_graph": round(ms1, 5),
            "algbw": round(alg, 2), "busbw": round(alg * (m - 1) / m, 2),
            "hbm_gbs": round(hbm / (ms * 1e-3) / 1e9, 1),
            "hbm_frac": round(hbm / (ms * 1e-3) / 1e9 / PEAK, 4)}


def sizes(lo, hi, step):
    s = lo
    while s <= hi:
        yield s
        s *= step


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "sweep.json"))
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    step = 16 if args.quick else 4
    rows = []

    def log(r):
        rows.append(r)
        print(json.dumps(r), flush=True)

    t0 = time.time()
    # config 1: the paper's 3-GPU fully connected example (DGX-1P {0,1,3})
    tri, _ = OG.induced(OG.dgx1p(), [0, 1, 3])
    comms = B.init_all([0] * 3, graph=B.Graph.from_pairs(3, tri[1]))
    for S in sizes(1 << 10, 1 << 30, step):
        log(run_coll(comms, "broadcast", S, "f32", 0, "c1-3gpu-triangle"))
        log(run_coll(comms, "allreduce", S, "f32", 0, "c1-3gpu-triangle"))
    for c in comms:
        c.destroy()
    # config 2: emulated DGX-1V, Broadcast from root 0 (6 ILP trees)
    g = OG.dgx1v()
    comms = B.init_all([0] * 8, graph=B.Graph.from_pairs(8, g[1]))
    for S in sizes(1 << 10, 1 << 30, step):
        log(run_coll(comms, "broadcast", S, "f32", 0, "c2-dgx1v-emulated"))
    for S in sizes(1 << 20, 1 << 28, 16):
        log(run_coll(comms, "allreduce", S, "f32", 0, "c2-dgx1v-emulated"))
    for c in comms:
        c.destroy()
    # config 3: 8-rank switch, one-hop AllReduce fp32 / bf16 (+ switch Broadcast)
    comms = B.init_all([0] * 8)
    for dt in ("f32", "bf16"):
        for S in sizes(1 << 10, 1 << 30, step):
            log(run_coll(comms, "allreduce", S, dt, 0, "c3-switch-onehop"))
    for S in sizes(1 << 10, 1 << 30, step):
        log(run_coll(comms, "broadcast", S, "f32", 0, "c3-switch"))
    # NEXT-3 duals on the same one-hop trees (S = bytes per rank of the full buffer)
    for S in sizes(1 << 16, 1 << 30, step * 4):
        for coll in ("reduce_scatter", "allgather"):
            log(run_block(comms, coll, S, "f32", "c3-switch-next3"))
    for c in comms:
        c.destroy()
    # config 4: fragmented allocations, re-packed
    for m in (3, 5, 6, 7):
        comms = B.init_all([0] * m)
        for S in sizes(1 << 10, 1 << 30, step * 4):
            log(run_coll(comms, "allreduce", S, "f32", 0, f"c4-switch-m{m}"))
        for c in comms:
            c.destroy()
    for nodes in ([0, 1, 4], [0, 1, 3, 4, 5, 7], [1, 4, 5, 6]):
        sub, _ = OG.induced(g, nodes)
        comms = B.init_all([0] * len(nodes), graph=B.Graph.from_pairs(len(nodes), sub[1]))
        log(run_coll(comms, "allreduce", 64 << 20, "f32", 0, f"c4-dgx1v-{''.join(map(str, nodes))}"))
        for c in comms:
            c.destroy()
    # NEXT-4: three-phase multi-server AllReduce, 3+5 and 4+4 emulated servers
    for servers in ([[0, 1, 3], [2, 4, 5, 6, 7]], [[0, 1, 2, 3], [4, 5, 6, 7]]):
        comms = B.init_all([0] * 8, graph=B.Graph.multi_server(8, g[1], servers))
        tag = "next4-" + "+".join(str(len(s)) for s in servers)
        for S in sizes(1 << 20, 1 << 28, 16):
            log(run_coll(comms, "allreduce", S, "f32", 0, tag))
        for c in comms:
            c.destroy()
    # config 5: DDP bucket sequences (App. C) at m = 2, 4, 8
    for m in (2, 4, 8):
        comms = B.init_all([0] * m)
        for (model, dt), buckets in synth.BUCKETS.items():
            bufs = [[torch.randn(n, device="cuda").to(TD[dt]) for _ in range(m)] for n in buckets]

            def seq():
                for bb in bufs:
                    for r, c in enumerate(comms):
                        c.allreduce(bb[r], bb[r])
            tot = sum(buckets) * ES[dt]
            ms, _ = time_calls(seq, tot)
            alg = tot / (ms * 1e-3) / 1e9
            log({"config": f"c5-{model}-buckets", "coll": "allreduce", "m": m, "dtype": dt,
                 "bytes": tot, "buckets": len(buckets), "ms": round(ms, 4), "algbw": round(alg, 2),
                 "busbw": round(alg * 2 * (m - 1) / m, 2),
                 "hbm_gbs": round(2 * m * tot / (ms * 1e-3) / 1e9, 1),
                 "hbm_frac": round(2 * m * tot / (ms * 1e-3) / 1e9 / PEAK, 4)})
            del bufs
        for c in comms:
            c.destroy()
    json.dump({"peak_hbm_gbs": PEAK, "device": torch.cuda.get_device_name(0), "rows": rows,
               "seconds": round(time.time() - t0, 1)}, open(args.out, "w"), indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
