#!/bin/bash
# parity (GPU tests) + device timings of cfg4 and cfg5 (64 profiles); ENVS="A=1;B=2" adds variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
IFS=';' read -ra SETS <<< "${ENVS:-X=0}"
for st in "${SETS[@]}"; do
  echo "[$st] $(env $st timeout 300 python scripts/dp_time.py cfg4 5) | $(env $st timeout 300 python scripts/dp_time.py cfg5 3)"
done
