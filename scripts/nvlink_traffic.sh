#!/bin/bash
# NVLink traffic evidence for the N > 1 bench: ncu in
# application-replay mode over every rank of a torchrun bench run, the NVLink
# transmit/receive byte counters of the Blink kernels, per launch, written to
# profiles/traffic.json under the bench workload key that bench.py reads
# (roofline.traffic).  Needs a multi-GPU box; one ncu call per size.
#
#   bash scripts/nvlink_traffic.sh 8 67108864     # N GPUs, fp32 elements per rank (256 MiB)
#
# Report: measured NVLink bytes / algorithmic bytes (AllReduce: 2(m-1)/m * S
# per GPU each way) and bytes / duration against 900 GB/s.
set -eu
N=${1:-8}
COUNT=${2:-67108864}
O=gpurun_out/nvlink
mkdir -p $O
ncu --replay-mode application --target-processes all --clock-control none \
    -k regex:exec_kernel --metrics nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum \
    --csv --log-file $O/nvl_${N}_${COUNT}.csv \
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
        bench.py --gpus $N --steps 2 --warmup 3 --count $COUNT --no-cpu-baseline > $O/bench_under_ncu_${N}.log 2>&1
python - "$O/nvl_${N}_${COUNT}.csv" "$N" "$COUNT" <<'PY'
import csv, json, os, sys
path, n, count = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
per = {}
for r in rows:
    k = (r.get("ID"), r.get("Process ID"))
    per.setdefault(k, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
tx = [v.get("nvltx__bytes_data_user.sum", 0.0) for v in per.values()]
rx = [v.get("nvlrx__bytes_data_user.sum", 0.0) for v in per.values()]
S = count * 4
alg = 2 * (n - 1) / n * S
mean_tx = sum(tx) / max(1, len(tx))
mean_rx = sum(rx) / max(1, len(rx))
key = f"c3-onehop-allreduce-m{n}-nvswitch-f32-{S >> 20}MiB"
tp = "profiles/traffic.json"
d = json.load(open(tp)) if os.path.exists(tp) else {}
d[key] = mean_tx + mean_rx
json.dump(d, open(tp, "w"), indent=1)
print(json.dumps({"workload": key, "launches": len(per), "nvl_tx_per_launch": mean_tx,
                  "nvl_rx_per_launch": mean_rx, "algorithmic_each_way": alg,
                  "tx_over_alg": mean_tx / alg if alg else None}))
PY
