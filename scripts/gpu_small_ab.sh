#!/bin/bash
# parity + k_fin small-cell A/B: dp_time for OOB_DP_SMALLPAIRS values on cfg5 (64 profiles) and cfg4
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for sp in ${PAIRS:-1 2 4 8 16}; do
  for si in 1 0; do
    echo "pairs=$sp seedinit=$si $(OOB_DP_SMALLPAIRS=$sp OOB_DP_SEEDINIT=$si timeout 300 python scripts/dp_time.py cfg5 3) | $(OOB_DP_SMALLPAIRS=$sp OOB_DP_SEEDINIT=$si timeout 300 python scripts/dp_time.py cfg4 3)"
  done
done
