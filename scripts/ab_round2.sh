#!/bin/bash
# Round-2 A/B: the shared-memory ring size (1 vs 2 co-resident CTAs per SM)
# on channel-heavy plans, and the shallow DGX-1V Broadcast trees.
mkdir -p gpurun_out/ab
for kb in 200 100 72; do
  BLINK_SMEM_KB=$kb CFG_LABEL=smem$kb timeout 600 python scripts/ab_bcast.py
done > gpurun_out/ab/ab_smem.txt 2>&1
cat gpurun_out/ab/ab_smem.txt
