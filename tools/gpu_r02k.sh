cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02k_build.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for v in main g6 gc64s3 gc16s8 gc48s4; do
  if [ $v = main ]; then L=""; else L="HPZ_LIB=$PWD/abtest_$v/libhpz.so"; fi
  env $L timeout 600 $B > gpurun_out/r02k_ab_$v.json 2> gpurun_out/r02k_ab_$v.err; echo "ab $v rc=$?"
done
CMD="python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/r02k_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file gpurun_out/r02k_launches_n1.csv $CMD > gpurun_out/r02k_ncu_launches.log 2>&1
echo "launches rc=$?"
SMALL="python bench.py --model falcon7b_block --steps 2 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 300 $SMALL > gpurun_out/r02k_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_tma_kernel|gather_tma_kernel" -s 3 -c 3 -o gpurun_out/r02k_prof_n1 $SMALL > gpurun_out/r02k_ncu_full.log 2>&1
echo "full rc=$?"
