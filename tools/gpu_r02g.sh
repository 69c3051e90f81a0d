cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02g_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -q -x -k "fingerprint or captured or special or ring or fused" > gpurun_out/r02g_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for v in main st10 st8; do
  if [ $v = main ]; then L=""; else L="HPZ_LIB=$PWD/abtest_$v/libhpz.so"; fi
  env $L timeout 600 $B > gpurun_out/r02g_bench_$v.json 2> gpurun_out/r02g_bench_$v.err; echo "bench $v rc=$?"
  env $L timeout 600 $B --verify none > gpurun_out/r02g_bench_${v}_nov.json 2> gpurun_out/r02g_bench_${v}_nov.err; echo "bench $v nov rc=$?"
done
SMALL="python bench.py --model falcon7b_block --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --graph 0"
timeout 300 $SMALL > gpurun_out/r02g_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_tma_kernel" -s 1 -c 1 -o gpurun_out/r02g_prof_fp $SMALL > gpurun_out/r02g_ncu_fp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_tma_kernel" -s 1 -c 1 -o gpurun_out/r02g_prof_nov $SMALL --verify none > gpurun_out/r02g_ncu_nov.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r02g_tests.log
