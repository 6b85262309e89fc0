#!/bin/bash
# A/B of environment knobs on the bench workload: ./scripts/ab_bench.sh "ENV=a" "ENV=b" ...
for cfg in "$@"; do
  for rep in 1 2 3; do
    v=$(env $cfg python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys;d=json.loads(sys.stdin.read());print(d['value'], d['roofline']['frac'])")
    echo "$cfg rep$rep: $v"
  done
done
