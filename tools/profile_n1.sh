#!/bin/bash
# ncu evidence for the N=1 bench (run under gpurun; one GPU).
set -x
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$?
$CMD > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"adam_kernel|gather_kernel|rs_kernel" -s 80 -c 6 -o gpurun_out/prof_n1 $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
