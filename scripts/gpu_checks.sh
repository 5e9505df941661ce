#!/bin/bash
# GPU validation: full gpu test suite, compute-sanitizer memcheck/racecheck on small configs,
# ncu DRAM traffic of every k_wave_w launch of one cfg4 template set.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in cfg2 cfg3; do
  timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python scripts/dp_once.py $c 1 > gpurun_out/memcheck_$c.log 2>&1; echo memcheck_$c=$?
  tail -2 gpurun_out/memcheck_$c.log
done
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/dp_once.py cfg2 1 > gpurun_out/racecheck_cfg2.log 2>&1; echo racecheck_cfg2=$?
tail -2 gpurun_out/racecheck_cfg2.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k 'regex:^k_wave_w' --csv --log-file gpurun_out/traffic_cfg4.csv python scripts/dp_once.py cfg4 1 > gpurun_out/ncu_traffic.log 2>&1; echo traffic=$?
