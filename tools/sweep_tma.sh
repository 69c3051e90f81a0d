#!/bin/bash
# gather TMA geometry sweep at N=$1 (run under gpurun --gpus N)
N=$1
for cfg in 32768,4,1 49152,4,1 65536,3,1 16384,6,2 32768,3,2 24576,4,2 16384,4,3; do
  timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus $N --steps 5 --no-e2e --no-cpu-baseline --no-nccl --tma $cfg > gpurun_out/sw.log 2>&1
  echo "$cfg $(grep -o 'breakdown[^}]*' gpurun_out/sw.log)"
done
