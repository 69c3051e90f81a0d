#!/bin/bash
# BASELINE north_star sweep: every model shape at N = 1, 2, 4 (one bench line each, NCCL
# baseline at N > 1).  Lines go to gpurun_out/sweep_<model>_n<N>.json.
cd "$(dirname "$0")/.."
run() { m=$1; n=$2; shift 2
  out=gpurun_out/sweep_${m}_n${n}.json
  if [ $n = 1 ]; then
    timeout 600 python bench.py --model $m --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $out.log 2>&1
  else
    timeout 600 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) \
      bench.py --gpus $n --model $m --steps 10 --warmup 3 --no-e2e --no-cpu-baseline "$@" > $out.log 2>&1
  fi
  rc=$?; tail -1 $out.log > $out; echo "$m n=$n rc=$rc"
}
for n in 1 2 4; do
  run falcon7b $n
  run llama2_7b $n
  run falcon40b_block $n
  run llama2_70b_layers $n
done
run llama2_13b 2 --grad-slots 2
run llama2_13b 4 --grad-slots 2
