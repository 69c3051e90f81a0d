cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02l_build.log 2>&1
B4="python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl"
B1="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for v in main gc16 gc8 wl wlgc16 pdl; do
  if [ $v = main ]; then L=""; else L="HPZ_LIB=$PWD/abtest_$v/libhpz.so"; fi
  env $L timeout 600 $B4 > gpurun_out/r02l_n4_$v.json 2> gpurun_out/r02l_n4_$v.err; echo "n4 $v rc=$?"
  env $L timeout 600 $B1 > gpurun_out/r02l_n1_$v.json 2> gpurun_out/r02l_n1_$v.err; echo "n1 $v rc=$?"
done
timeout 600 python bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02l_bench_n4_full.json 2> gpurun_out/r02l_bench_n4_full.err; echo "full n4 rc=$?"
