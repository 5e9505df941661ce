#!/bin/bash
# A/B timing of an alternative build of the library (build/lib_*.so) against the in-tree one.
mkdir -p gpurun_out
for v in ${VARIANTS}; do
  cp paper_2309_08125_b200/liboobleck_plan.so /tmp/lib_main.so
  cp build/lib_$v.so paper_2309_08125_b200/liboobleck_plan.so
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  tail -1 gpurun_out/ab_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step'], d['roofline']['frac'])"
  cp /tmp/lib_main.so paper_2309_08125_b200/liboobleck_plan.so
done
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ab_main.log 2>&1
tail -1 gpurun_out/ab_main.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('main', d['ms_per_step'], d['roofline']['frac'])"
