#!/bin/bash
# ncu --set full of k_fin at chosen wavefronts (skip count) of a config (default cfg5, 64 profiles)
CFG=${CFG:-cfg5}
NP=${NP:-64}
mkdir -p gpurun_out
python scripts/dp_once.py $CFG 1 $NP > gpurun_out/plain.log 2>&1 || { echo plain-failed; cat gpurun_out/plain.log; exit 1; }
for s in ${WAVES:-24}; do
  OOB_DP_SEEDINIT=${SEEDINIT:-1} timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_fin' -s $s -c 1 -o gpurun_out/prof_fin_${CFG}_s$s python scripts/dp_once.py $CFG 1 $NP > gpurun_out/ncu_fin_s$s.log 2>&1; echo full_s$s=$?
done
