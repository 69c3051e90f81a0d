# A/B: gather CTAs rotating through sources (HPZ_GATHER_ROTATE=1, main) vs pinned (abtest_norot)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02aa_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/r02aa_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02aa_tests.log
for n in 4 2 1; do
  B="python bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
  for v in main norot main2 norot2; do
    case $v in main|main2) L="";; *) L="HPZ_LIB=$PWD/abtest_norot/libhpz.so";; esac
    env $L timeout 600 $B > gpurun_out/r02aa_n${n}_$v.json 2> gpurun_out/r02aa_n${n}_$v.err; echo "n$n $v rc=$?"
  done
done
