#!/bin/bash
# per-wave timelines of cfg5 (and cfg4) under plan-time switches (run under gpurun)
mkdir -p gpurun_out
OOB_NVCC_DEFS="OOB_TIMELINE" python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > /dev/null
i=0
for ENV in "$@"; do
  i=$((i+1))
  echo "== [$ENV]" > gpurun_out/tl_cfg5_$i.txt
  env $ENV python scripts/timeline.py cfg5 1 >> gpurun_out/tl_cfg5_$i.txt 2>&1
done
python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > /dev/null
