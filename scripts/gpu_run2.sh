set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1; echo bench=$?
tail -2 gpurun_out/bench_cfg4.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --workload cfg5 > gpurun_out/bench_cfg5.log 2>&1; echo bench5=$?
tail -2 gpurun_out/bench_cfg5.log
