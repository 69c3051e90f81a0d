#!/bin/bash
# ncu evidence for the N=1 bench (run under gpurun; one GPU).
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file gpurun_out/launches_n1.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo launches_rc=$?
ncu --set full --clock-control none --import-source on -k regex:"rs_tma_kernel|gather_tma_kernel" -s 40 -c 4 -o gpurun_out/prof_n1 $CMD > gpurun_out/ncu_full.log 2>&1
echo full_rc=$?
