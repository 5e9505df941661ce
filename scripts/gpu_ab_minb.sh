#!/bin/bash
# A/B of k_wave_w's resident-CTA target (OOB_WAVE_MINB) on cfg4/cfg5: per-wave timelines and
# step times (run under gpurun).
mkdir -p gpurun_out
for MB in ${@:-2 3}; do
  OOB_NVCC_DEFS="OOB_WAVE_MINB=$MB OOB_TIMELINE" python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > /dev/null
  python scripts/timeline.py cfg4 3 > gpurun_out/timeline_cfg4_mb$MB.txt 2>&1
  OOB_NVCC_DEFS="OOB_WAVE_MINB=$MB" python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > /dev/null
  echo "MINB=$MB" >> gpurun_out/ab_minb.txt
  python scripts/dp_time.py cfg4 20 >> gpurun_out/ab_minb.txt 2>&1
  python scripts/dp_time.py cfg5 3 >> gpurun_out/ab_minb.txt 2>&1
done
python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > /dev/null
