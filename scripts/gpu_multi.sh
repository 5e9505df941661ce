#!/bin/bash
# N-GPU bench (torchrun, one rank per GPU, NCCL): cfg4 (independent per-rank profiles) and cfg5 (sharded sweep).
mkdir -p gpurun_out
N=${N:-2}
for wl in cfg4 cfg5; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $N --steps 3 --warmup 3 --workload $wl > gpurun_out/bench_${wl}_n$N.log 2>&1; echo bench_${wl}_n$N=$?
  tail -1 gpurun_out/bench_${wl}_n$N.log | cut -c1-300
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29535 \
  bench.py --gpus $N --steps 5 --warmup 3 --shard-profile > gpurun_out/bench_cfg4_shard_n$N.log 2>&1; echo bench_cfg4_shard_n$N=$?
tail -1 gpurun_out/bench_cfg4_shard_n$N.log | cut -c1-400
