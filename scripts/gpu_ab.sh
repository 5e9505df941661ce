#!/bin/bash
# A/B timing (scripts/dp_time.py) of alternative builds build/lib_<v>.so against the in-tree library.
mkdir -p gpurun_out
cp paper_2309_08125_b200/liboobleck_plan.so /tmp/lib_main.so
for v in ${VARIANTS}; do
  cp build/lib_$v.so paper_2309_08125_b200/liboobleck_plan.so
  echo -n "$v: "; timeout 300 python scripts/dp_time.py ${WL:-cfg4} 5 2>&1 | tail -1
  cp /tmp/lib_main.so paper_2309_08125_b200/liboobleck_plan.so
done
echo -n "main: "; timeout 300 python scripts/dp_time.py ${WL:-cfg4} 5 2>&1 | tail -1
