#!/bin/bash
# Round-2 GPU evidence: -m gpu suite, the three sanitizers (full logs), A/B of
# deferred chunk signals on the multi-hop Broadcast / AllReduce configs, and
# the chunk-pipelining fit.  Output under gpurun_out/$1/.
O=gpurun_out/${1:-r2}
mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q > $O/gputest.log 2>&1; echo "pytest rc=$?" >> $O/gputest.log
for t in memcheck synccheck racecheck; do
  echo "=== compute-sanitizer --tool $t python scripts/sanitize_cases.py"
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_cases.py 2>&1
  echo "=== exit $?"
done > $O/sanitizer.txt
for d in 0 1 0 1; do BLINK_DEFER_SIGNAL=$d CFG_LABEL=defer$d timeout 600 python scripts/ab_bcast.py; done > $O/ab_defer.txt 2>&1
timeout 900 python scripts/pipeline_model.py --out $O/pipeline.json > $O/pipeline.log 2>&1
tail -3 $O/gputest.log; grep -E "^ok|sanitize cases ok|SUMMARY|=== |MISMATCH|WRONG|Error" $O/sanitizer.txt; cat $O/ab_defer.txt; tail -5 $O/pipeline.log
