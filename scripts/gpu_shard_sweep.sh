#!/bin/bash
# 4-GPU single-profile sharding sweep over plan switches (run under gpurun --gpus 4):
#   bash scripts/gpu_shard_sweep.sh "OOB_DP_SHARDMIN=2000000" "OOB_DP_FINHELP=1024" ...
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null
N=${N:-4}
i=0
for E in "$@"; do
  i=$((i+1))
  env $E timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29700 + i)) scripts/shard_check.py cfg4 20 > gpurun_out/sweep_$i.log 2>&1
  echo "[$E] $(grep -o '"ms_per_template_set[^,]*' gpurun_out/sweep_$i.log) $(grep -o 'identical[^]]*' gpurun_out/sweep_$i.log)"
done
