#!/bin/bash
# ncu --set full of k_wave_w at chosen wavefronts of cfg4 (skip count = l - 2); CFG selects the W config.
mkdir -p gpurun_out
[ -n "$CFG" ] && export OOB_DP_WCFG=$CFG
python scripts/dp_once.py cfg4 1 > gpurun_out/plain.log 2>&1 || { echo plain-failed; cat gpurun_out/plain.log; exit 1; }
for s in ${WAVES:-30 78}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_wave_w' -s $s -c 1 -o gpurun_out/prof_w${CFG}_s$s python scripts/dp_once.py cfg4 1 > gpurun_out/ncu_full_s$s.log 2>&1; echo full_s$s=$?
done
