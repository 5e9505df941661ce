#!/bin/bash
# A/B of env settings on the cfg4 bench: VARIANTS="A=1 B=2;C=3" (';'-separated sets)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
IFS=';' read -ra VS <<< "${VARIANTS:-}"
for v in "" "${VS[@]}"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCHARGS} > gpurun_out/ab.log 2>&1
  tail -1 gpurun_out/ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[$v]', 'ms', round(d['ms_per_step'],3), 'frac', round(d['roofline']['frac'],4))" 2>&1 | tail -1
done
