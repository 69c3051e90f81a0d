#!/bin/bash
# ncu evidence for the N=1 bench (run under gpurun; one GPU).
#  1) launch list of the bench command itself (one pass per kernel, no replay)
#  2) --set full of one launch of each hot kernel on a small arena (one Falcon-7B decoder
#     block, the size of the bench's decoder-layer launches):
#     kernel replay saves/restores device memory, which is slow on the 166 GB bench arena
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$?
SMALL="python bench.py --model falcon7b_block --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $SMALL > gpurun_out/prof_plain_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_tma_kernel|gather_tma_kernel" -s 3 -c 3 -o gpurun_out/prof_n1 $SMALL > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
