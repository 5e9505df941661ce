#!/bin/bash
# single-profile sharding (bench.py --shard-profile) on N GPUs under plan-time switches
# (run under gpurun --gpus N):  bash scripts/gpu_shard_ab.sh N "ENV=.." ...
N=$1; shift
mkdir -p gpurun_out
port=29600
for ENV in "$@"; do
  port=$((port+1))
  echo "[$ENV] N=$N" >> gpurun_out/shard_ab.txt
  env $ENV timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N --steps 10 --warmup 3 --shard-profile --no-cpu-baseline > gpurun_out/shard_tmp.json 2>>gpurun_out/shard_ab.err
  python -c "import json; d=json.loads(open('gpurun_out/shard_tmp.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['e2e']['planning_latency_ms'])" >> gpurun_out/shard_ab.txt 2>&1
done
