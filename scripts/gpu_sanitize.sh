#!/bin/bash
# compute-sanitizer passes (memcheck, racecheck, synccheck, initcheck) over small template
# sets through the device path (run under gpurun); summaries to gpurun_out/sanitize_*.txt
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
for tool in memcheck racecheck synccheck initcheck; do
  for cfg in cfg2 cfg3; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/dp_time.py $cfg 1 \
        > gpurun_out/sanitize_${tool}_${cfg}.txt 2>&1
    echo "$tool $cfg rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|error' gpurun_out/sanitize_${tool}_${cfg}.txt | tail -1)"
  done
done
