mkdir -p gpurun_out/ab
for i in 1 2; do CFG_LABEL=new$i timeout 600 python scripts/ab_bcast.py; done > gpurun_out/ab/ab_ticket.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_per_rank.py -q -x > gpurun_out/ab/tests.log 2>&1; tail -2 gpurun_out/ab/tests.log
cat gpurun_out/ab/ab_ticket.txt
