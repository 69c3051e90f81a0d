cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02y_build.log 2>&1
HPZ_LIB=$PWD/abtest_rcp/libhpz.so timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_fuzz.py -q -x > gpurun_out/r02y_rcp_tests.log 2>&1; echo "rcp tests rc=$?"
B="python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e"
for v in main rcp main2 rcp2; do
  case $v in main|main2) L="";; *) L="HPZ_LIB=$PWD/abtest_rcp/libhpz.so";; esac
  env $L timeout 600 $B > gpurun_out/r02y_$v.json 2> gpurun_out/r02y_$v.err; echo "$v rc=$?"
  env $L timeout 600 $B --verify none > gpurun_out/r02y_${v}_nov.json 2> gpurun_out/r02y_${v}_nov.err; echo "$v nov rc=$?"
done
tail -3 gpurun_out/r02y_rcp_tests.log
