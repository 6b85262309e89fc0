#!/bin/bash
# Round-2 A/B: chunk floor of multi-hop trees after the deferred signals
# (BLINK_DEEP_CAP caps the bytes/16 floor; default 96 KiB link graphs, 64 KiB switch).
mkdir -p gpurun_out/ab
for cap in 16384 32768 65536 98304 0; do
  if [ $cap = 0 ]; then lab=default; export -n BLINK_DEEP_CAP; unset BLINK_DEEP_CAP; else lab=cap$cap; export BLINK_DEEP_CAP=$cap; fi
  CFG_LABEL=$lab timeout 600 python scripts/ab_bcast.py
done > gpurun_out/ab/ab_deepcap.txt 2>&1
unset BLINK_DEEP_CAP
for mc in 4096 8192 16384; do
  BLINK_MIN_CHUNK_DEEP=$mc CFG_LABEL=mcd$mc timeout 600 python scripts/ab_bcast.py
done >> gpurun_out/ab/ab_deepcap.txt 2>&1
cat gpurun_out/ab/ab_deepcap.txt
