# local gathers by the wide kernel + remote gathers in counter order (main) vs wide + static
# remote order (static) vs the previous kernels (old); parity suites first
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ax_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py tests/test_gpu_stock_schedule.py tests/test_gpu_multiproc.py tests/test_gpu_multiproc_shared.py -m gpu -x -q > gpurun_out/r02ax_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02ax_tests.log
for n in 1 4 2; do
  B="python bench.py --gpus $n --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
  for v in main static old; do
    case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
    env $L timeout 600 $B > gpurun_out/r02ax_n${n}_$v.json 2> gpurun_out/r02ax_n${n}_$v.err; echo "n$n $v rc=$?"
  done
done
