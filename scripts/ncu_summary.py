#!/usr/bin/env python
"""Summarise ncu outputs into committed files under profiles/.

    python scripts/ncu_summary.py --rep gpurun_out/prof.ncu-rep --launches gpurun_out/launches.csv \
        --tag r01 --workload c3-onehop-allreduce-m8-virtual-1gpu-f32-256MiB

Writes profiles/ncu_<tag>_summary.json (key metrics of the captured kernel,
stall reasons, launch-list shares) and updates profiles/traffic.json
(dram bytes per launch of the dominant kernel, read by bench.py).
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit)
    return float(v) * mult if mult else None


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u = rows[0], rows[1]
    kernels = []
    for v in rows[2:]:
        d = {h[i]: (v[i], u[i]) for i in range(len(h)) if i < len(v)}
        kernels.append(d)
    return kernels


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(list)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            name = r[ki]
            short = name.split("(")[0].replace("void ", "")[:80]
            agg[short].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    return {k: {"launches": len(v), "mean_ns": sum(v) / len(v), "share": sum(v) / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--tag", required=True)
    ap.add_argument("--workload", required=True)
    ap.add_argument("--kernel", default="exec_kernel")
    args = ap.parse_args()
    summ = {"tag": args.tag, "workload": args.workload}
    if args.rep:
        ks = [k for k in raw(args.rep) if args.kernel in k.get("Kernel Name", ("", ""))[0]]
        k = ks[0]
        summ["kernel"] = k["Kernel Name"][0]
        summ["metrics"] = {m: {"value": k[m][0], "unit": k[m][1]} for m in KEYS if m in k}
        stalls = {}
        for m, (val, _) in k.items():
            if m.startswith("smsp__pcsamp_warps_issue_stalled_") and not m.endswith("not_issued"):
                try:
                    if float(val) > 0:
                        stalls[m.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(val)
                except ValueError:
                    pass
        tot = sum(stalls.values()) or 1
        summ["stall_share"] = {s: round(v / tot, 4) for s, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:10]}
        rd = to_bytes(*k["dram__bytes_read.sum"])
        wr = to_bytes(*k["dram__bytes_write.sum"])
        summ["dram_bytes_per_launch"] = rd + wr
        tpath = os.path.join(ROOT, "profiles", "traffic.json")
        t = json.load(open(tpath)) if os.path.exists(tpath) else {}
        t[args.workload] = rd + wr
        json.dump(t, open(tpath, "w"), indent=1, sort_keys=True)
    if args.launches:
        summ["launch_list"] = launches(args.launches)
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    out = os.path.join(ROOT, "profiles", f"ncu_{args.tag}_summary.json")
    json.dump(summ, open(out, "w"), indent=1)
    print(out)


if __name__ == "__main__":
    main()
