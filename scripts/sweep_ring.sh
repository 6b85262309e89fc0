#!/bin/bash
# tuning sweep of the TMA ring (run under gpurun)
for thr in 256 512; do for smem in 108 200 224; do for tile in 0 2048 8192; do
  if [ $thr = 512 ] && [ $smem = 108 ]; then continue; fi
  r=$(BLINK_SMEM_KB=$smem BLINK_TILE=$tile BLINK_THREADS=$thr timeout 120 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['roofline']['frac'], d['roofline']['kernel_ms'])" 2>&1)
  echo "thr=$thr smem=$smem tile=$tile -> $r"
done; done; done
