#!/bin/bash
# W-kernel tile-width A/B: dp_time per forced OOB_DP_WCFG (0: TE4, 1: TE5, 2: TE3, 3: TE2) and auto over all
mkdir -p gpurun_out
for c in ${CFGS:-0 2 3}; do
  echo "wcfg=$c $(OOB_DP_WCFG=$c timeout 300 python scripts/dp_time.py cfg5 3) | $(OOB_DP_WCFG=$c timeout 300 python scripts/dp_time.py cfg4 3)"
done
echo "auto4 $(OOB_DP_AUTOCFGS=4 timeout 300 python scripts/dp_time.py cfg5 3) | $(OOB_DP_AUTOCFGS=4 timeout 300 python scripts/dp_time.py cfg4 3)"
