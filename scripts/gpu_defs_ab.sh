#!/bin/bash
# rebuild with diagnostic defines (DEFS="A B;C" sets) and run a parity subset (K=pytest -k expr)
mkdir -p gpurun_out
IFS=';' read -ra SETS <<< "${DEFS:-NONE}"
for st in "${SETS[@]}"; do
  OOB_NVCC_DEFS="$st" python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > gpurun_out/build_defs.log 2>&1 || { echo build-failed; tail gpurun_out/build_defs.log; }
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${K:-cfg1 or cfg2}" 2>&1 | tail -1 | sed "s/^/[$st] /"
done
