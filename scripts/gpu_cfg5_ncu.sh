#!/bin/bash
# cfg5 (1024 random 48-layer profiles, one set) on one GPU (run under gpurun): bench line,
# ncu launch list, DRAM traffic per k_wave_w launch, full captures of waves 12 and 36.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --workload cfg5 --steps 3 --warmup 3 > gpurun_out/c5_bench.json 2> gpurun_out/c5_bench.err
timeout 300 python scripts/dp_time.py cfg5 1 1024 > gpurun_out/c5_dptime.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c5_launches.csv \
    python scripts/dp_time.py cfg5 1 1024 > /dev/null 2>&1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
    -k regex:k_wave_w --launch-skip 141 --launch-count 47 --log-file gpurun_out/c5_traffic.csv \
    python scripts/dp_time.py cfg5 1 1024 > /dev/null 2>&1
for W in 12 36; do
  ncu --set full --import-source on --clock-control none -k regex:k_wave_w --launch-skip $((141 + W - 2)) \
      --launch-count 1 -o gpurun_out/c5_ncu_wave$W -f python scripts/dp_time.py cfg5 1 1024 > gpurun_out/c5_ncu_wave$W.log 2>&1
done
tail -c 400 gpurun_out/c5_bench.json; cat gpurun_out/c5_dptime.txt
