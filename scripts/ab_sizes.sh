#!/bin/bash
# A/B of env knobs at several sizes (device time of graph replays, m=8 one-hop AllReduce)
for cfg in "$@"; do
  env $cfg python - <<'PY'
import os, torch, sys
sys.path.insert(0, os.getcwd())
import paper_1910_04940_b200 as B
comms = B.init_all([0] * 8)
out = []
for nbytes in (1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20):
    cnt = nbytes // 4
    xs = [torch.randn(cnt, device="cuda") for _ in range(8)]
    ys = [torch.empty_like(x) for x in xs]
    def fn():
        for r, c in enumerate(comms):
            c.allreduce(xs[r], ys[r])
    for _ in range(3): fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g): fn()
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / reps * 1e3
    out.append(f"{nbytes>>20}MiB:{us:.1f}us/{nbytes/us/1e3:.0f}GB/s")
print(os.environ.get("CFG_LABEL", ""), " ".join(out), flush=True)
PY
  echo "   ^ $cfg"
done
