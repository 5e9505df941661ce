#!/bin/bash
# Round artefacts: gpu tests, cfg4 bench (with cpu_baseline), cfg5 bench, reference arm,
# ncu launch list of the bench command, ncu --set full of one large k_wave_w launch, traffic.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -20 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_cfg4.log 2>&1; echo bench4=$?; tail -1 gpurun_out/bench_cfg4.log | cut -c1-200
timeout 600 python bench.py --workload cfg5 --steps 3 --no-cpu-baseline > gpurun_out/bench_cfg5.log 2>&1; echo bench5=$?; tail -1 gpurun_out/bench_cfg5.log | cut -c1-200
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k 'regex:^k_wave_w' --csv --log-file gpurun_out/traffic_cfg4.csv python scripts/dp_once.py cfg4 1 > gpurun_out/ncu_traffic.log 2>&1; echo traffic=$?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_wave_w" -s 78 -c 1 -f -o gpurun_out/prof_final_w80 python scripts/dp_once.py cfg4 1 > gpurun_out/ncu_full.log 2>&1; echo full=$?
ncu -i gpurun_out/prof_final_w80.ncu-rep --page raw --csv > gpurun_out/prof_final_w80.raw.csv 2>&1
ncu -i gpurun_out/prof_final_w80.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_final_w80.sass.csv 2>&1
