cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02s_build.log 2>&1
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for v in main p1c2 l12 l24k; do
  if [ $v = main ]; then L=""; else L="HPZ_LIB=$PWD/abtest_$v/libhpz.so"; fi
  env $L timeout 600 $B > gpurun_out/r02s_$v.json 2> gpurun_out/r02s_$v.err; echo "$v rc=$?"
  env $L timeout 600 $B --verify none > gpurun_out/r02s_${v}_nov.json 2> gpurun_out/r02s_${v}_nov.err; echo "$v nov rc=$?"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "missing_peer or checkpoint" > gpurun_out/r02s_tests.log 2>&1; echo "tests rc=$?"
