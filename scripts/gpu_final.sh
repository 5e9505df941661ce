#!/bin/bash
# Round measurements on one GPU (run under gpurun): GPU tests, bench lines (cfg4, cfg5,
# reference arm), ncu launch list + DRAM traffic of one cfg4 set, full captures of two waves,
# exact-solver timings.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_pytest_gpu.log 2>&1; tail -3 gpurun_out/final_pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/final_bench_cfg4.json 2> gpurun_out/final_bench_cfg4.err
timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 3 > gpurun_out/final_bench_cfg5.json 2> gpurun_out/final_bench_cfg5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_cfg4.csv \
    python scripts/dp_time.py cfg4 1 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:k_wave_w --launch-skip 95 --launch-count 95 --log-file gpurun_out/final_traffic_cfg4.csv \
    python scripts/dp_time.py cfg4 1 > /dev/null 2>&1
for W in 36 80; do
  ncu --set full --import-source on --clock-control none -k regex:k_wave_w --launch-skip $((95 + W - 2)) \
      --launch-count 1 -o gpurun_out/final_ncu_wave$W -f python scripts/dp_time.py cfg4 1 > gpurun_out/final_ncu_wave$W.log 2>&1
done
tail -c 300 gpurun_out/final_bench_cfg4.json
for c in "cfg2 5" "cfg3 3" "cfg4 3" "cfg5 1 64"; do timeout 300 python scripts/exact_time.py $c; done > gpurun_out/final_exact_time.txt 2>&1
