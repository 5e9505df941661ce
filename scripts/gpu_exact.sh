mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q > gpurun_out/ex_pytest.log 2>&1; tail -15 gpurun_out/ex_pytest.log
for c in "cfg2 5" "cfg3 3" "cfg4 2" "cfg5 1 64"; do timeout 300 python scripts/exact_time.py $c; done 2>&1 | tee gpurun_out/ex_time.txt
