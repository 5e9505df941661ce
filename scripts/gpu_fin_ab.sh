#!/bin/bash
# k_fin / seeding A/B on a config (default cfg5, 64 profiles): dp_time plus ncu launch-list totals per kernel
CFG=${CFG:-cfg5}
NP=${NP:-64}
mkdir -p gpurun_out
for si in 1 0; do
  echo "== SEEDINIT=$si"
  OOB_DP_SEEDINIT=$si timeout 300 python scripts/dp_time.py $CFG 3
  OOB_DP_SEEDINIT=$si timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
     --log-file gpurun_out/fin_ab_${CFG}_si$si.csv python scripts/dp_once.py $CFG 1 $NP > /dev/null 2>&1
done
