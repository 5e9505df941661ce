#!/bin/bash
# Quick GPU iteration: parity tests (fail fast), cfg4 bench per W-kernel config, launch list.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu.log
for c in ${CFGS:-auto 0 1}; do
  if [ $c = auto ]; then unset OOB_DP_WCFG; else export OOB_DP_WCFG=$c; fi
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_$c.log 2>&1; echo bench4_$c=$?
  tail -1 gpurun_out/bench_cfg4_$c.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms_per_step'], d['e2e']['planning_latency_ms'])" 2>&1 | tail -2
done
unset OOB_DP_WCFG
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches.csv python scripts/dp_once.py cfg4 1 > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
python scripts/wave_table.py gpurun_out/launches.csv | head -8
