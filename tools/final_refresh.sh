#!/bin/bash
# End-of-round evidence on one box (gpurun --gpus 4): ncu captures first (their traffic
# feeds the bench lines), then the bench lines at N = 1, 2, 4, the oracle reference arm,
# smoke(), and the f3 transformer run at a communication-heavier size.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('SMOKE_OK')" > gpurun_out/fr_smoke.log 2>&1; echo "smoke rc=$?"
bash tools/profile_n1.sh
python tools/ncu_summary.py gpurun_out/prof_n1.ncu-rep > gpurun_out/fr_ncu_summary.log 2>&1; echo "ncu_summary rc=$?"
cp profiles/ncu_traffic.json profiles/r01_ncu_full_n1_final.csv gpurun_out/
cp gpurun_out/launches_n1.csv gpurun_out/r01_ncu_launches_n1_final.csv 2>/dev/null
timeout 600 python bench.py > gpurun_out/fr_n1.log 2>&1; echo "bench n1 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fr_ref_n1.log 2>&1; echo "ref rc=$?"
for n in 2 4; do
  timeout 900 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2950$n bench.py --gpus $n > gpurun_out/fr_n$n.log 2>&1; echo "bench n$n rc=$?"
done
TF="--model transformer --h 4096 --heads 32 --ffn 11008 --seq 1024 --tokens 1024 --layers 8 --steps 8 --warmup 2 --max-ctas 32 --lr 1e-5"
for n in 2 4; do
  timeout 900 torchrun --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n tools/train_overlap.py $TF > gpurun_out/fr_f3tf1k_n$n.log 2>&1; echo "f3 n$n rc=$?"
done
