#!/bin/bash
# One GPU validation pass: gpu parity tests, bench (cfg4, cfg5), ncu launch list + one full capture.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1; nproc >> gpurun_out/lscpu.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_cfg4.log 2>&1; echo bench4=$?
tail -1 gpurun_out/bench_cfg4.log | cut -c1-600
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload cfg5 > gpurun_out/bench_cfg5.log 2>&1; echo bench5=$?
tail -1 gpurun_out/bench_cfg5.log | cut -c1-400
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^k_wave_w' -s 78 -c 1 -o gpurun_out/prof_w python scripts/dp_once.py cfg4 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
