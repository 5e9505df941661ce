#!/bin/bash
# A/B of environment switches on the cfg4 bench: ENVS="A=1 B=0;C=1" (';'-separated settings)
mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "${ENVS}"
for st in "${SETS[@]}"; do
  env $st timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/envab.log 2>&1
  tail -1 gpurun_out/envab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$st]', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))" 2>&1 | tail -1
done
