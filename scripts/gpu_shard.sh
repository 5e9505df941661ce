#!/bin/bash
# Single-profile sharding check on N GPUs (and N=1 through the same path).
mkdir -p gpurun_out
N=${N:-2}
for n in 1 $N; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29541 \
    scripts/shard_check.py cfg4 5 > gpurun_out/shard_n$n.log 2>&1; echo shard_n$n=$?
  grep workload gpurun_out/shard_n$n.log || tail -5 gpurun_out/shard_n$n.log
done
