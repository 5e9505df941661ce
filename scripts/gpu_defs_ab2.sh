#!/bin/bash
# A/B of compile-time variants: DEFS="A=1;A=0 B=2" (';'-separated OOB_NVCC_DEFS sets), cfg4 (and BENCHARGS) bench.
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${DEFS:-}"
for v in "${VS[@]}"; do
  OOB_NVCC_DEFS="$v" python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > gpurun_out/build_ab.log 2>&1 || { tail -5 gpurun_out/build_ab.log; continue; }
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCHARGS} > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4))" 2>&1 | tail -1
done
