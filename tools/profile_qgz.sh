#!/bin/bash
# ncu --set full of one qgZ quantize launch on a small arena (one Falcon-40B block, N=1).
CMD="python bench.py --model falcon40b_block --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --qgz"
timeout 300 $CMD > gpurun_out/pq_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"qgz_quantize" -s 1 -c 1 -o gpurun_out/prof_qgz $CMD > gpurun_out/pq_ncu.log 2>&1
echo rc=$?
