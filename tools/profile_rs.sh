#!/bin/bash
# ncu --set full of one fused RS+Adam launch on a small arena (one Falcon-40B block, N=1).
CMD="python bench.py --model falcon40b_block --steps 2 --warmup 1 --no-e2e --no-cpu-baseline $EXTRA"
timeout 300 $CMD > gpurun_out/prs_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_tma_kernel" -s 1 -c 1 -o gpurun_out/prof_rs $CMD > gpurun_out/prs_ncu.log 2>&1
echo rc=$?
