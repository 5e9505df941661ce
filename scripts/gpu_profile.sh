#!/bin/bash
# GPU-box diagnostics (run under gpurun): timeline build + per-wave timeline, then the
# normal build, an ncu launch list and one --set full capture of chosen wavefronts.
#   gpurun -- bash scripts/gpu_profile.sh [waves...]   (default waves: 24 48 80)
set -x
mkdir -p gpurun_out
OOB_NVCC_DEFS=OOB_TIMELINE python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)"
python scripts/timeline.py cfg4 3 > gpurun_out/timeline_cfg4.txt 2>&1
python scripts/timeline.py cfg5 1 > gpurun_out/timeline_cfg5.txt 2>&1
python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)"
python scripts/dp_time.py cfg4 20 > gpurun_out/dp_time_cfg4.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv \
    python scripts/dp_time.py cfg4 1 > /dev/null 2>&1
for W in ${@:-24 48 80}; do
  # launch index of wave W among k_wave_w launches: warm-up run + timed run(s); capture one
  ncu --set full --import-source on --clock-control none -k regex:k_wave_w --launch-skip $((W - 2)) \
      --launch-count 1 -o gpurun_out/ncu_wave$W -f python scripts/dp_time.py cfg4 1 > gpurun_out/ncu_wave$W.log 2>&1
done
