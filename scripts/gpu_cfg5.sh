#!/bin/bash
# cfg5 (1024-profile batched sweep) step time under plan-time switches (run under gpurun)
mkdir -p gpurun_out
for ENV in "$@"; do
  echo "[$ENV]" >> gpurun_out/cfg5_ab.txt
  env $ENV python bench.py --workload cfg5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_tmp.json 2>>gpurun_out/cfg5_ab.txt
  python -c "import json; d=json.loads(open('gpurun_out/cfg5_tmp.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['roofline']['frac'], d['e2e']['planning_latency_ms'])" >> gpurun_out/cfg5_ab.txt
done
