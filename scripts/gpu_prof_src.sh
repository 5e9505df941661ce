#!/bin/bash
# ncu source-level capture of k_wave_w at wave l = S+2 (WAVES="78 30"), SASS csv + raw metrics.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
python scripts/dp_once.py ${CFG:-cfg4} 1 > gpurun_out/plain.log 2>&1 || { cat gpurun_out/plain.log; exit 1; }
for s in ${WAVES:-78}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_wave_w' -s $s -c 1 -f -o gpurun_out/src_s$s python scripts/dp_once.py ${CFG:-cfg4} 1 > gpurun_out/ncu_src_s$s.log 2>&1; echo full_s$s=$?
  ncu -i gpurun_out/src_s$s.ncu-rep --page source --csv --print-source sass > gpurun_out/src_s$s.sass.csv 2>&1
  ncu -i gpurun_out/src_s$s.ncu-rep --page raw --csv > gpurun_out/src_s$s.raw.csv 2>&1
done
