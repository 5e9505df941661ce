#!/bin/bash
# Parity tests, one bench line, and an ncu source-level (SASS) capture of k_wave_w at wave l = S+2.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log
for s in ${WAVES:-78}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_wave_w' -s $s -c 1 -o gpurun_out/src_s$s python scripts/dp_once.py cfg4 1 > gpurun_out/ncu_src_s$s.log 2>&1; echo full_s$s=$?
  ncu -i gpurun_out/src_s$s.ncu-rep --page source --csv --print-source sass > gpurun_out/src_s$s.sass.csv 2>&1; echo src=$?
done
