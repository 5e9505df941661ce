#!/bin/bash
# Single-profile sharding A/B over OOB_DP_SHARDMIN at N GPUs (torchrun).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
N=${N:-4}
for sm in ${SMS:-2e7 5e7 1e8 2e8}; do
  OOB_DP_SHARDMIN=$sm timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29561 \
    bench.py --gpus $N --steps 5 --warmup 3 --shard-profile --no-cpu-baseline > gpurun_out/shard_ab.log 2>&1
  tail -1 gpurun_out/shard_ab.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('[shardmin $sm]', 'ms', round(d['ms_per_step'],3))" 2>&1 | tail -1
done
