set -u
for n in 2 3 4; do
  for base in 1000 2000; do
    MODE=fuzz BLINK_SAME_GPU=1 MP_FUZZ_N=25 MP_FUZZ_BASE=$((base + n * 100)) PYTHONPATH=. timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29600 + n * 10 + base / 1000)) tests/mp_worker.py 2>&1 | grep -E "fuzz ok|mismatch|Error|error" | head -5
  done
done
