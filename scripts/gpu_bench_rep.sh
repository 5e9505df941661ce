#!/bin/bash
# Repeat the cfg4 bench R times (run-to-run variance on one box).
mkdir -p gpurun_out
for i in $(seq 1 ${R:-3}); do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_rep_$i.log 2>&1
  tail -1 gpurun_out/bench_rep_$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$i', d['ms_per_step'], d['roofline']['frac'], d['clocks'])"
done
