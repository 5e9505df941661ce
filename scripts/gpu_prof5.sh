mkdir -p gpurun_out
export OOB_DP_WCFG=1
python scripts/dp_once.py cfg4 1 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k 'regex:^k_wave_w$' -s 78 -c 1 -o gpurun_out/prof_w80 python scripts/dp_once.py cfg4 1 > gpurun_out/ncu2.log 2>&1
echo full=$?
