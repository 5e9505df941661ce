mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu.log
for c in auto 0 1 2 3; do
  if [ $c = auto ]; then unset OOB_DP_WCFG; else export OOB_DP_WCFG=$c; fi
  timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_$c.log 2>&1; echo bench_$c=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_cfg4_$c.log').read().strip().splitlines()[-1]);print('$c', d['ms_per_step'], d['roofline']['frac'])"
done
for c in auto 0 2; do
  if [ $c = auto ]; then unset OOB_DP_WCFG; else export OOB_DP_WCFG=$c; fi
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload cfg5 > gpurun_out/bench_cfg5_$c.log 2>&1; echo bench5=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_cfg5_$c.log').read().strip().splitlines()[-1]);print('cfg5 $c', d['ms_per_step'], d['roofline']['frac'])"
done
