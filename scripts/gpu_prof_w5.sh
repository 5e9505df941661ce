#!/bin/bash
# ncu --set full of k_wave_w at chosen wavefronts (skip count = l - 2) of cfg5 (64 profiles)
mkdir -p gpurun_out
python scripts/dp_once.py cfg5 1 64 > gpurun_out/plain.log 2>&1 || { echo plain-failed; cat gpurun_out/plain.log; exit 1; }
for s in ${WAVES:-23}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:k_wave_w' -s $s -c 1 -o gpurun_out/prof_w5${WCFG}_s$s python scripts/dp_once.py cfg5 1 64 > gpurun_out/ncu_w5_s$s.log 2>&1; echo full_s$s=$?
done
