#!/bin/bash
# A/B of plan-time switches on cfg4/cfg5 step time (run under gpurun):
#   bash scripts/gpu_ab_env.sh "" "OOB_DP_FINWAIT=0" ...
mkdir -p gpurun_out
for ENV in "$@"; do
  for rep in 1 2; do
    echo "[$ENV] rep $rep" >> gpurun_out/ab_env.txt
    env $ENV python scripts/dp_time.py cfg4 20 >> gpurun_out/ab_env.txt 2>&1
  done
  env $ENV python scripts/dp_time.py cfg5 3 >> gpurun_out/ab_env.txt 2>&1
done
