#!/bin/bash
# Quick iteration: build, cfg4 golden parity (fused default), bench line, flush stats build.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "${PYK:-cfg4_full_vs_golden and default or configs_vs_oracle}" > gpurun_out/pytest_quick.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_quick.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCHARGS} > gpurun_out/bench.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ms', d['ms_per_step'], 'frac', d['roofline']['frac'], 'kernel_ms', d['roofline']['kernel_ms_per_step'])"
if [ -n "$STATS" ]; then
  OOB_FLUSH_STATS=1 python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
  python scripts/flush_stats.py cfg4
  python -c "from paper_2309_08125_b200 import build as b; b.build(force=True)" > /dev/null 2>&1
fi
