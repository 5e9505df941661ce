#!/bin/bash
# Multi-GPU bench lines (run under gpurun --gpus N): weak cfg4 (one profile per rank),
# cfg4 single-profile sharding (peer exchange), cfg5 1024-profile sweep (strong)
N=${1:-4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
run() {  # name, port, args...
  local name=$1 port=$2; shift 2
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N "$@" > gpurun_out/multi_${name}_n$N.json 2> gpurun_out/multi_${name}_n$N.err
  tail -c 250 gpurun_out/multi_${name}_n$N.json
}
run cfg4 29701 --steps 20 --warmup 5
run cfg4_shard 29702 --steps 20 --warmup 5 --shard-profile
run cfg5 29703 --workload cfg5 --steps 3 --warmup 3
