#!/bin/bash
# per-wave k_wave_w times (ncu launch list) for forced tile widths on cfg4 and cfg5 (64 profiles)
mkdir -p gpurun_out
for c in ${CFGS:-0 2}; do
  for k in cfg4 cfg5; do
    OOB_DP_WCFG=$c timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/tew_${k}_$c.csv python scripts/dp_once.py $k 1 > /dev/null 2>&1; echo $k $c $?
  done
done
