#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python scripts/dbg_parity.py real
OOB_DP_SEEDINIT=0 python scripts/dbg_parity.py real
OOB_DP_FUSE=0 python scripts/dbg_parity.py real
OOB_DP_WCFG=3 python scripts/dbg_parity.py real
OOB_DP_WCFG=2 python scripts/dbg_parity.py real
python scripts/dbg_parity.py dyadic
