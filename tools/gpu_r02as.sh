# gather chunks from a per-launch counter (HPZ_GATHER_DYN=1, main) vs static grid-stride (static)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02as_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_stock_schedule.py -m gpu -x -q > gpurun_out/r02as_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02as_tests.log
B="python bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for r in 1 2; do
  for v in main static; do
    case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
    env $L timeout 300 $B > gpurun_out/r02as_${v}_$r.json 2> gpurun_out/r02as_${v}_$r.err; echo "$v $r rc=$?"
  done
done
