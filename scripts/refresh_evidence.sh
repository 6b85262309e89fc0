#!/bin/bash
# One GPU call that regenerates the round's evidence under gpurun_out/ev/:
# bench line, ncu launch list of the bench command, ncu --set full captures of
# the bench kernel and of the DGX-1V multi-hop Broadcast kernel, sweep,
# per-rank sweep, pipeline fit, sanitizer (full logs).  Summarise locally with
# scripts/ncu_summary.py and copy into profiles/ (named per round).
set -u
O=gpurun_out/ev
mkdir -p $O
python bench.py > $O/bench.json 2> $O/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 2 -c 1 -o $O/prof \
    python scripts/one_call.py 8 268435456 f32 ar 3 > $O/ncu_full.log 2>&1
ONE_CALL_GRAPH=dgx1v ncu --set full --clock-control none --import-source on -k regex:exec_kernel -s 2 -c 1 \
    -o $O/prof_dgx1v_bc python scripts/one_call.py 8 67108864 f32 bc 3 > $O/ncu_dgx1v.log 2>&1
python scripts/sweep.py --out $O/sweep.json > $O/sweep.log 2>&1
python scripts/per_rank_sweep.py --out $O/per_rank_sweep.json > $O/per_rank_sweep.log 2>&1 || true
python scripts/pipeline_model.py --out $O/pipeline.json > $O/pipeline.log 2>&1 || true
# full logs (no tail: the round-1 logs hid a failing script behind `tail -3`)
for t in memcheck synccheck racecheck; do
  echo "=== compute-sanitizer --tool $t python scripts/sanitize_cases.py"
  timeout 1200 compute-sanitizer --tool $t python scripts/sanitize_cases.py 2>&1
  echo "=== exit $?"
done > $O/sanitizer.txt
echo done
