#!/usr/bin/env python
"""Benchmark: tree-packed AllReduce (Blink, arXiv:1910.04940) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl blink|reference]

Workload (BASELINE.json configs[2], "8xB200 NVSwitch one-hop-tree AllReduce"):
AllReduce SUM of S = 256 MiB fp32 per rank over m = 8 ranks planned as m
one-hop trees.  One step = one whole AllReduce (split, reduce to
each tree root, broadcast back) = one launch of the tree executor.

* N = 1 (default): the 8 ranks are virtual ranks on cuda:0 -- all 8 ranks'
  buffers live in this GPU's HBM and one cooperative launch runs every rank's
  channels (the same kernels/tables as the multi-GPU path; the fabric is HBM,
  so the roofline is HBM bandwidth).
* N > 1 (torchrun): one process per GPU, m = N real ranks over NVLink/NVSwitch
  with symmetric registered buffers (CUDA IPC); handles exchanged over gloo.

metric = algBW = S / t (GB/s, per-rank buffer bytes per collective time, the
nccl-tests convention); busBW = algBW * 2(m-1)/m is reported alongside.
Inputs: 8 x 256 MiB = 2 GiB per step, larger than the 126 MB L2 (no flush).
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DEFAULT_M = 8
DEFAULT_COUNT = 64 << 20           # 256 MiB fp32 per rank
METRIC = "AllReduce/Broadcast algBW GB/s vs size, 2/4/8 B200, % NVLink peak vs NCCL"
REF_SAMPLE_COUNT = 4 << 20         # oracle samples (cpu_baseline and --impl reference): 16 MiB fp32 per rank
UNIT = "GB/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0}, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
         "utilization.gpu")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "10"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return None
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                util = float(parts[9]) if len(parts) > 9 else 100.0
                rows.append(dict(sm=float(parts[1]), smax=float(parts[2]), hw=parts[5], hwt=parts[6],
                                 swt=parts[7], pcap=parts[8], util=util, pw=float(parts[3])))
            except ValueError:
                continue
        if not rows:
            return None
        # every sample falls inside the timed region (the sampler starts 0.3 s
        # before it); nvidia-smi's utilization / power are slow running
        # averages, so they are reported but not used to select samples
        busy = rows
        reasons = set()
        for r in rows:
            for k, name in (("hw", "hw_slowdown"), ("hwt", "hw_thermal_slowdown"),
                            ("swt", "sw_thermal_slowdown"), ("pcap", "sw_power_cap")):
                if r[k].lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(r["sm"] for r in rows),
                "sm_max_mhz": max(r["smax"] for r in rows), "reasons": sorted(reasons),
                "samples": len(rows), "max_power_w": max(r["pw"] for r in rows),
                "note": "10 ms nvidia-smi samples spanning the timed region"}


def cpu_oracle_baseline(m, count, budget_s=10.0, max_s=30.0):
    """The oracle (oracle/, plain numpy, single-threaded) on a bounded sample of
    the same workload: AllReduce of `count` fp32 per rank over m one-hop trees,
    repeated until ~budget_s of CPU time."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import synth
    from oracle import collectives as OC
    from oracle import packing as OP
    plan = OP.plan_switch_allreduce(m)
    sends = synth.inputs(3, m, count, "f32")
    reps, t = 0, 0.0
    while t < budget_s and reps < 100:
        t0 = time.perf_counter()
        OC.allreduce(plan, sends, "f32", "sum")
        t += time.perf_counter() - t0
        reps += 1
        if t > max_s:
            break
    value = reps * count * 4 / t / 1e9
    return {"value": round(value, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{reps} x AllReduce of {count} fp32/rank over {m} one-hop trees "
                      f"({count * 4 >> 20} MiB/rank), numpy single-thread, {t:.1f}s",
            "host_cpus": os.cpu_count()}


def traffic_from_profiles(workload):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(p)).get(workload)
    except Exception:
        return None


# --------------------------------------------------------------------------- blink arm
def run_virtual(args):
    import torch
    import synth
    import paper_1910_04940_b200 as B

    m, count, dtype = args.ranks, args.count, "f32"
    S = count * 4
    comms = B.init_all([0] * m, cfg=B.config(timeout_s=60.0))
    sends = [synth.device_input(3, r, count, dtype) for r in range(m)]
    recvs = [torch.empty_like(s) for s in sends]
    stream = torch.cuda.current_stream()

    def step():
        for r, c in enumerate(comms):
            c.allreduce(sends[r], recvs[r], op="sum", stream=stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches0 = comms[0].stats()["launches"]
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with Clocks(0) as clk:
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for k in range(args.steps):
            starts[k].record(stream)
            step()
            ends[k].record(stream)
        t1.record(stream)
        torch.cuda.synchronize()
    launches = comms[0].stats()["launches"] - launches0
    ms = t0.elapsed_time(t1) / args.steps
    kern_ms = statistics.mean(s.elapsed_time(e) for s, e in zip(starts, ends))
    algbw = S / (ms * 1e-3) / 1e9

    # e2e: the same call with HOST buffers.  Every step copies every rank's
    # input H2D from pinned memory, runs the collective, and copies every
    # rank's result D2H into pinned memory -- all inside the timed region.
    # Results are double-buffered so step k's D2H (copy stream) overlaps step
    # k+1's H2D (compute stream).
    hsend = [s.cpu().pin_memory() for s in sends]
    hrecv = [[torch.empty(count, dtype=torch.float32).pin_memory() for _ in range(m)] for _ in range(2)]
    recv2 = [recvs, [torch.empty_like(s) for s in sends]]
    d2h = torch.cuda.Stream()
    ev_free = [None, None]
    # 20 steps (or K if fewer): the first step's H2D and the last step's D2H
    # run alone (pipeline fill / drain), every other step overlaps them
    # (scripts/pcie_probe.py: 2.15 GB each way concurrently in 43 ms)
    e2e_steps = max(2, min(args.steps, 20))

    def e2e_step(k):
        i = k % 2
        for r in range(m):
            sends[r].copy_(hsend[r], non_blocking=True)
        if ev_free[i] is not None:
            stream.wait_event(ev_free[i])
        for r, c in enumerate(comms):
            c.allreduce(sends[r], recv2[i][r], op="sum", stream=stream)
        done = torch.cuda.Event()
        done.record(stream)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            for r in range(m):
                hrecv[i][r].copy_(recv2[i][r], non_blocking=True)
        ev_free[i] = torch.cuda.Event()
        ev_free[i].record(d2h)

    e2e_step(0)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(e2e_steps):
        e2e_step(k)
    stream.wait_stream(d2h)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / e2e_steps

    peaks, how = load_peaks()
    workload = arm_config(m, S, 1)["workload"]
    alg_bytes = 2 * m * S        # HBM: read every rank's send once, write every rank's recv once
    achieved = alg_bytes / (kern_ms * 1e-3) / 1e9
    peak = float(peaks["hbm_gbs"])
    out = {
        "metric": METRIC, "value": round(algbw, 3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded N(0,1)*1e-2 gradients, generated on device)",
        "config": arm_config(m, S, 1),
        "bus_bw_gbs": round(algbw * 2 * (m - 1) / m, 3),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic_from_profiles(workload),
                     "peak_source": f"{how} hbm_gbs",
                     "algorithmic_bytes_per_launch": alg_bytes, "kernel_ms": round(kern_ms, 4)},
        "e2e": {"value": round(S / (e2e_ms * 1e-3) / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": m * S, "d2h_bytes_per_step": m * S,
                "ms_per_step": round(e2e_ms, 3),
                "steps": e2e_steps,
                "note": "every rank's input H2D and result D2H (pinned) per step; D2H of step k overlaps H2D of step k+1"},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    out["protocol_path"] = per_rank_protocol(B, m, sends, recvs, S, stream, max(3, min(args.steps, 20)))
    out["vs_size"] = size_profile(torch, comms, sends, recvs)
    if not args.no_cpu_baseline:   # the same sample as the reference arm: 16 MiB per rank
        out["cpu_baseline"] = cpu_oracle_baseline(m, min(count, REF_SAMPLE_COUNT))
    for c in comms:
        c.destroy()
    return out


def size_profile(torch, comms, sends, recvs, sizes=(1 << 10, 64 << 10, 1 << 20, 16 << 20, 64 << 20)):
    """The metric is "algBW vs size": AllReduce and Broadcast (root 0) on the
    same m virtual ranks at a few sizes per rank, device time per call of 10
    back-to-back calls captured in one CUDA graph (a graph launch costs ~2 us
    of its own), algBW = S / t.  Context for the headline, which is the
    256 MiB AllReduce above; sizes up to 1 MiB stay in the 126 MB L2 across
    replays (profiles/sweep_r02.json has every config)."""
    out = {"note": "per-call device time, 10 calls per CUDA graph, m virtual ranks; sizes with 2*m*S <= 126 MB "
                   "stay L2-resident across replays", "allreduce": {}, "broadcast": {}}
    for coll in ("allreduce", "broadcast"):
        for nb in sizes:
            cnt = nb // 4

            def call():
                for r, c in enumerate(comms):
                    if coll == "allreduce":
                        c.allreduce(sends[r][:cnt], recvs[r][:cnt], op="sum")
                    else:
                        c.broadcast(sends[0][:cnt] if r == 0 else None, recvs[r][:cnt], root=0)
            for _ in range(3):
                call()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                for _ in range(10):
                    call()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                g.replay()
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) / 50 * 1e3
            key = f"{nb >> 20} MiB" if nb >= (1 << 20) else f"{nb >> 10} KiB"
            out[coll][key] = {"us": round(us, 2), "alg_bw_gbs": round(nb / (us * 1e-6) / 1e9, 2)}
            del g
    return out


NVLINK_GBS = 900.0   # NVLink 5 per direction per B200 (busBW / 900)


class Nccl:
    """NCCL 2.28 (torch's bundled libnccl) called directly through ctypes: the
    comparison the metric names, on the SAME device buffers and stream as
    Blink, out of place, AllReduce and Broadcast, eager and CUDA-graph
    captured; optionally with symmetric-window registration (ncclMemAlloc +
    ncclCommWindowRegister, NCCL_WIN_COLL_SYMMETRIC).  NCCL is never on
    Blink's data path."""
    FLOAT32, SUM = 7, 0

    def __init__(self, rank, world):
        import ctypes
        import glob
        import torch.distributed as dist
        import nvidia
        base = os.path.dirname(list(nvidia.__path__)[0])
        cands = glob.glob(os.path.join(base, "nvidia", "nccl", "lib", "libnccl.so*"))
        if not cands:
            raise RuntimeError("libnccl.so not found")
        self.lib = ctypes.CDLL(cands[0])
        self.ct = ctypes

        class UID(ctypes.Structure):
            _fields_ = [("internal", ctypes.c_char * 128)]
        uid = UID()
        if rank == 0:
            self._ok(self.lib.ncclGetUniqueId(ctypes.byref(uid)), "ncclGetUniqueId")
        obj = [bytes(uid.internal) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid.internal = obj[0]
        self.comm = ctypes.c_void_p()
        self._ok(self.lib.ncclCommInitRank(ctypes.byref(self.comm), world, uid, rank), "ncclCommInitRank")
        v = ctypes.c_int()
        self.lib.ncclGetVersion(ctypes.byref(v))
        self.version = v.value

    def _ok(self, r, what):
        if r != 0:
            raise RuntimeError(f"{what} returned {r}")

    def allreduce(self, send, recv, count, stream):
        self._ok(self.lib.ncclAllReduce(self.ct.c_void_p(send), self.ct.c_void_p(recv), self.ct.c_size_t(count),
                                        self.FLOAT32, self.SUM, self.comm, self.ct.c_void_p(stream)),
                 "ncclAllReduce")

    def broadcast(self, send, recv, count, root, stream):
        self._ok(self.lib.ncclBroadcast(self.ct.c_void_p(send), self.ct.c_void_p(recv), self.ct.c_size_t(count),
                                        self.FLOAT32, root, self.comm, self.ct.c_void_p(stream)),
                 "ncclBroadcast")

    def mem_alloc(self, nbytes):
        p = self.ct.c_void_p()
        self._ok(self.lib.ncclMemAlloc(self.ct.byref(p), self.ct.c_size_t(nbytes)), "ncclMemAlloc")
        return p.value

    def window(self, ptr, nbytes):
        w = self.ct.c_void_p()
        self._ok(self.lib.ncclCommWindowRegister(self.comm, self.ct.c_void_p(ptr), self.ct.c_size_t(nbytes),
                                                 self.ct.byref(w), 1), "ncclCommWindowRegister")
        return w

    def close(self):
        self.lib.ncclCommDestroy(self.comm)


def tuning_lines(path):
    """NCCL's algorithm/protocol choices from its NCCL_DEBUG=INFO TUNING log."""
    out = []
    try:
        for line in open(path):
            low = line.lower()
            if ("algo" in low or "protocol" in low or "proto" in low) and ("allreduce" in low or "broadcast" in low):
                txt = line.strip().split("NCCL INFO", 1)[-1].strip()
                if txt not in out:
                    out.append(txt)
            if len(out) >= 6:
                break
    except OSError:
        pass
    return out


def time_device(fn, steps, stream, graph=False):
    """Mean ms per call over `steps` calls with CUDA events on `stream`
    (eager), or of one CUDA graph holding `steps` calls, replayed once."""
    import torch
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    if graph:
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()           # captures need a non-default stream
        cs.wait_stream(stream)
        with torch.cuda.graph(g, stream=cs):
            for _ in range(steps):
                fn()
        g.replay()
        torch.cuda.synchronize()
        t0.record(stream)
        g.replay()
        t1.record(stream)
    else:
        t0.record(stream)
        for _ in range(steps):
            fn()
        t1.record(stream)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1) / steps


def multiprocess_line(args, m, S, ms, bc_ms, graph, e2e_ms, n_e2e, launches, clocks, nccl):
    """Rank 0's JSON line at N > 1 (pure: tested on the CPU with given times).
    AllReduce is the headline (`value` = algBW); busBW = algBW * 2(m-1)/m is
    measured against NVLink's 900 GB/s per direction; the
    Broadcast arm (busBW = algBW) and NCCL's numbers ride along."""
    workload = arm_config(m, S, m)["workload"]
    algbw = S / (ms * 1e-3) / 1e9
    bus = algbw * 2 * (m - 1) / m
    bc_alg = S / (bc_ms * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": round(algbw, 3), "unit": UNIT, "n_gpus": m,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded N(0,1)*1e-2 gradients, generated on device)",
        "config": arm_config(m, S, m),
        "bus_bw_gbs": round(bus, 3),
        "roofline": {"bound": "nvlink", "achieved": round(bus, 2), "peak": NVLINK_GBS, "unit": "GB/s",
                     "frac": round(bus / NVLINK_GBS, 4),
                     "traffic": traffic_from_profiles(workload),
                     "peak_source": "NVLink 5 nominal per direction (SURVEY 8(d): busBW / 900); "
                                    "traffic: ncu nvltx+nvlrx bytes per launch from profiles/traffic.json "
                                    "(scripts/nvlink_traffic.sh), null until measured"},
        "broadcast": {"root": 0, "ms": round(bc_ms, 4), "alg_bw_gbs": round(bc_alg, 3),
                      "bus_bw_gbs": round(bc_alg, 3), "frac": round(bc_alg / NVLINK_GBS, 4)},
        "graph": graph,
        "e2e": {"value": round(S / (e2e_ms * 1e-3) / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": S, "d2h_bytes_per_step": S, "steps": n_e2e,
                "note": "per rank: input H2D and result D2H (pinned); D2H of step k overlaps H2D of step k+1"},
        "gpu_launches": launches, "clocks": clocks,
        "nccl": nccl,
    }
    return out


def per_rank_protocol(B, m, sends, recvs, S, stream, steps):
    """The same AllReduce with one launch per rank (cfg.launch_per_rank): the
    kernels and cross-launch protocol a real one-process-per-GPU rank runs
    (entry handshake, per-chunk flags between launches, exit waits), here with
    1/m of the SMs per rank.  The headline `value` times the single launch
    that holds every virtual rank (no flags); this shows what the protocol
    costs on the same bytes."""
    import torch
    comms = B.init_all([0] * m, cfg=B.config(timeout_s=60.0, launch_per_rank=1))

    def step():
        for r, c in enumerate(comms):
            c.allreduce(sends[r], recvs[r], op="sum", stream=stream)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(steps):
        step()
    t1.record(stream)
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / steps
    st = comms[0].stats()
    for c in comms:
        c.destroy()
    return {"ms_per_step": round(ms, 4), "alg_bw_gbs": round(S / (ms * 1e-3) / 1e9, 3), "steps": steps,
            "hbm_frac": round(2 * m * S / (ms * 1e-3) / 1e9 / float(load_peaks()[0]["hbm_gbs"]), 4),
            "launches_per_step": m, "ctas_per_launch": st["last_ctas"],
            "note": "launch_per_rank=1: one launch per rank with the multi-process protocol (entry "
                    "handshake, per-chunk flags, exit waits), 1/m of the SMs each"}


def run_multiprocess(args):
    import torch
    import torch.distributed as dist
    import synth
    import paper_1910_04940_b200 as B

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    same_gpu = os.environ.get("BENCH_SAME_GPU") == "1"   # test harness: all ranks share cuda:0
    if same_gpu:
        local = 0
    # NCCL reads its environment once, at its first communicator: set the
    # comparison's knobs before anything initialises it
    tune_log = os.path.join(tempfile.gettempdir(), f"bench_nccl_tuning.{os.getpid()}.log")
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "TUNING")
    os.environ["NCCL_DEBUG_FILE"] = tune_log
    if args.nccl_nvls is not None:
        os.environ["NCCL_NVLS_ENABLE"] = str(args.nccl_nvls)
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    ex = B.torch_exchange()
    comm = B.init_multiprocess(world, rank, local, ex, cfg=B.config(timeout_s=60.0))
    count = args.count
    S = count * 4
    send = synth.device_input(3, rank, count, "f32")
    recv = torch.empty_like(send)
    comm.register(send, S, ex)
    comm.register(recv, S, ex)
    stream = torch.cuda.current_stream()

    # calls enqueue on the current stream: `stream` eagerly, the capture
    # stream inside a CUDA-graph capture
    def blink_ar():
        comm.allreduce(send, recv, op="sum", stream=torch.cuda.current_stream())

    def blink_bc():
        comm.broadcast(send if rank == 0 else None, recv, root=0, count=count, dtype="f32",
                       stream=torch.cuda.current_stream())

    def max_ms(ms):
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        blink_ar()
        blink_bc()
    torch.cuda.synchronize()
    dist.barrier()
    launches0 = comm.stats()["launches"]
    with Clocks(local) as clk:
        torch.cuda.synchronize()
        dist.barrier()
        ms = time_device(blink_ar, args.steps, stream)
        dist.barrier()
    ms = max_ms(ms)
    launches = comm.stats()["launches"] - launches0
    dist.barrier()
    bc_ms = max_ms(time_device(blink_bc, args.steps, stream))
    dist.barrier()
    graph = {}
    try:
        graph["blink_allreduce_ms"] = round(max_ms(time_device(blink_ar, args.steps, stream, graph=True)), 4)
        dist.barrier()
        graph["blink_broadcast_ms"] = round(max_ms(time_device(blink_bc, args.steps, stream, graph=True)), 4)
    except Exception as e:  # pragma: no cover - depends on the box
        graph["blink_unavailable"] = f"{type(e).__name__}: {e}"[:160]
    m = world
    # e2e through host buffers (pinned): H2D input, collective, D2H result.
    # Results are double-buffered (a second registered recv) so step k's D2H
    # (copy stream) overlaps step k+1's H2D, as in the N = 1 line.
    hsend = send.cpu().pin_memory()
    recv2 = torch.empty_like(send)
    comm.register(recv2, S, ex)
    recvs = [recv, recv2]
    hrecvs = [torch.empty(count, dtype=torch.float32).pin_memory() for _ in range(2)]
    d2h = torch.cuda.Stream()
    ev_free = [None, None]

    def e2e_step(k):
        i = k % 2
        send.copy_(hsend, non_blocking=True)
        if ev_free[i] is not None:
            stream.wait_event(ev_free[i])
        comm.allreduce(send, recvs[i], op="sum", stream=stream)
        done = torch.cuda.Event()
        done.record(stream)
        d2h.wait_event(done)
        with torch.cuda.stream(d2h):
            hrecvs[i].copy_(recvs[i], non_blocking=True)
        ev_free[i] = torch.cuda.Event()
        ev_free[i].record(d2h)

    e2e_step(0)
    torch.cuda.synchronize()
    dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    n_e2e = max(2, min(args.steps, 20))
    for k in range(n_e2e):
        e2e_step(k)
    stream.wait_stream(d2h)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_ms(e0.elapsed_time(e1) / n_e2e)
    nccl = nccl_compare(args, send, recv, count, stream, rank, world, same_gpu, tune_log)
    nvls = nvls_arm(args, B, ex, send, count, stream, rank, world, max_ms) if not same_gpu else \
        {"unavailable": "all ranks share one GPU (a multicast team needs distinct GPUs)"}
    out = None
    if rank == 0:
        out = multiprocess_line(args, m, S, ms, bc_ms, graph, e2e_ms, n_e2e, launches, clk.summary(), nccl)
        out["nvls"] = nvls
    comm.destroy()
    dist.barrier()
    dist.destroy_process_group()
    return out


def nvls_arm(args, B, ex, send, count, stream, rank, world, max_ms):
    """NEXT-1 on the same workload: a second comm with cfg.nvls = 1 (the one-hop
    trees inside the NVSwitch).  Reports whether multicast came up (and why
    not), the AllReduce time, and the largest deviation from the P2P result
    relative to sum|x| (the switch sums in its own order, R#29).  Any failure
    is recorded, not raised: the P2P line stands on its own."""
    import torch
    import torch.distributed as dist
    out = {}
    comm = None
    try:
        comm = B.init_multiprocess(world, rank, torch.cuda.current_device(), ex,
                                   cfg=B.config(timeout_s=10.0, nvls=1))
        plan = comm.plan(True, 0, count, "f32")
        out["active"] = plan["nvls"]["active"]
        out["note"] = plan["nvls"]["note"]
        if out["active"]:
            ref = torch.empty_like(send)
            comm2 = B.init_multiprocess(world, rank, torch.cuda.current_device(), ex,
                                        cfg=B.config(timeout_s=10.0))
            comm2.allreduce(send, ref, op="sum", stream=stream)
            y = torch.empty_like(send)

            def arm():
                comm.allreduce(send, y, op="sum", stream=torch.cuda.current_stream())

            for _ in range(args.warmup):
                arm()
            torch.cuda.synchronize()
            dist.barrier()
            ms = max_ms(time_device(arm, args.steps, stream))
            S = count * 4
            alg = S / (ms * 1e-3) / 1e9
            dev = float((y - ref).abs().max()) / max(1e-30, float(send.abs().max()) * world)
            t = torch.tensor([dev], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out.update({"ms": round(ms, 4), "alg_bw_gbs": round(alg, 3),
                        "bus_bw_gbs": round(alg * 2 * (world - 1) / world, 3),
                        "max_dev_vs_p2p_rel": float(t.item())})
            comm2.destroy()
    except Exception as e:  # pragma: no cover - depends on the box
        out["error"] = f"{type(e).__name__}: {e}"[:200]
    finally:
        if comm is not None:
            try:
                comm.destroy()
            except Exception:
                pass
    return out


def nccl_compare(args, send, recv, count, stream, rank, world, same_gpu, tune_log):
    """NCCL on the same buffers, stream and step count, out of place, max over
    ranks: AllReduce and Broadcast, eager and CUDA-graph captured, and the
    symmetric-window variant; plus the algorithm / protocol NCCL chose."""
    import torch
    import torch.distributed as dist
    if same_gpu:
        return {"unavailable": "all ranks share one GPU (NCCL needs one GPU per rank)"}
    out = {}
    try:
        nc = Nccl(rank, world)
    except Exception as e:  # pragma: no cover - depends on the box
        return {"unavailable": f"{type(e).__name__}: {e}"[:200]}
    S = count * 4

    def max_ms(ms):
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def arm(name, fn, f_bus):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        ms = max_ms(time_device(fn, args.steps, stream))
        alg = S / (ms * 1e-3) / 1e9
        out[name] = {"ms": round(ms, 4), "alg_bw_gbs": round(alg, 3), "bus_bw_gbs": round(alg * f_bus, 3)}
        try:
            dist.barrier()
            gms = max_ms(time_device(fn, args.steps, stream, graph=True))
            out[name]["graph_ms"] = round(gms, 4)
        except Exception as e:  # pragma: no cover
            out[name]["graph"] = f"{type(e).__name__}"[:80]

    f_ar = 2 * (world - 1) / world
    sptr, rptr = send.data_ptr(), recv.data_ptr()

    def cur():
        return torch.cuda.current_stream().cuda_stream

    try:
        arm("allreduce", lambda: nc.allreduce(sptr, rptr, count, cur()), f_ar)
        arm("broadcast", lambda: nc.broadcast(sptr, rptr, count, 0, cur()), 1.0)
        try:   # symmetric windows (NCCL 2.27+): buffers from ncclMemAlloc
            a = nc.mem_alloc(S)
            b = nc.mem_alloc(S)
            torch.cuda.synchronize()
            nc.window(a, S)
            nc.window(b, S)
            arm("allreduce_symmetric", lambda: nc.allreduce(a, b, count, cur()), f_ar)
        except Exception as e:  # pragma: no cover
            out["allreduce_symmetric"] = {"unavailable": f"{type(e).__name__}: {e}"[:160]}
    except Exception as e:  # pragma: no cover - depends on the box
        out["error"] = f"{type(e).__name__}: {e}"[:200]
    torch.cuda.synchronize()
    out["impl"] = f"NCCL {nc.version} (ctypes, torch's libnccl), out of place, same buffers and stream"
    out["env"] = {k: os.environ[k] for k in ("NCCL_NVLS_ENABLE", "NCCL_ALGO", "NCCL_PROTO") if k in os.environ}
    out["tuning"] = tuning_lines(tune_log)
    nc.close()
    return out


# --------------------------------------------------------------------------- config
def arm_config(m, S, world):
    """The workload both arms report (`config`): the Blink arm runs it, the
    reference arm times a bounded sample of it (cpu_baseline.sample)."""
    if world > 1:
        return {"workload": f"c3-onehop-allreduce-m{m}-nvswitch-f32-{S >> 20}MiB", "collective": "allreduce",
                "op": "sum", "ranks": m, "ranks_kind": "one process per GPU", "bytes_per_rank": S,
                "l2": f"{2 * S >> 20} MiB send+recv per rank per step"
                      + (" > 126 MB L2" if 2 * S > (126 << 20) else " (fits L2)")}
    return {"workload": f"c3-onehop-allreduce-m{m}-virtual-1gpu-f32-{S >> 20}MiB", "collective": "allreduce",
            "op": "sum", "ranks": m, "ranks_kind": "virtual (all on cuda:0)", "bytes_per_rank": S,
            "trees": m, "plan": "one-hop stars (P:440-442)",
            "l2": f"send+recv {2 * m * S >> 30} GiB/step > 126 MB L2 (no flush needed)"
                  if 2 * m * S > (126 << 20) else "inputs fit L2"}


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as the reference arm (no reference implementation exists):
    rank 0 times oracle/ on a bounded sample of the same workload."""
    if int(os.environ.get("RANK", "0")) != 0:
        return None
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import synth
    from oracle import collectives as OC
    from oracle import packing as OP
    m = args.ranks if int(os.environ.get("WORLD_SIZE", "1")) == 1 else int(os.environ["WORLD_SIZE"])
    count = min(args.count, REF_SAMPLE_COUNT)
    plan = OP.plan_switch_allreduce(m)
    sends = synth.inputs(3, m, count, "f32")
    for _ in range(args.warmup):
        OC.allreduce(plan, sends, "f32", "sum")
    t0 = time.perf_counter()
    for _ in range(args.steps):
        OC.allreduce(plan, sends, "f32", "sum")
    t = (time.perf_counter() - t0) / args.steps
    v = count * 4 / t / 1e9
    world = int(os.environ.get("WORLD_SIZE", "1"))
    sample = (f"bounded sample of the workload: AllReduce of {count} fp32/rank ({count * 4 >> 20} MiB of the "
              f"{args.count * 4 >> 20} MiB per rank) over {m} one-hop trees per step, numpy single-thread")
    return {"metric": METRIC, "value": round(v, 4), "unit": UNIT, "impl": "reference",
            "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(t * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": arm_config(m, args.count * 4, world),
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": sample, "host_cpus": os.cpu_count()},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="blink", choices=["blink", "reference"])
    ap.add_argument("--ranks", type=int, default=DEFAULT_M, help="virtual ranks at N=1")
    ap.add_argument("--count", type=int, default=DEFAULT_COUNT, help="fp32 elements per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nccl-nvls", type=int, default=None, choices=[0, 1],
                    help="N>1: NCCL_NVLS_ENABLE for the NCCL comparison (set before NCCL initialises)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        out = run_reference(args)
    elif int(os.environ.get("WORLD_SIZE", "1")) > 1:
        out = run_multiprocess(args)
    else:
        out = run_virtual(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
