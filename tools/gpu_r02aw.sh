# gather: dynamic chunk order with the counter read ahead + unrolled fingerprint warps (main, runs of 4 chunks per counter update), g2, g8,
# (g2, g8: runs of 2 / 8 chunks), static order (static); fingerprint on / off
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02aw_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/r02aw_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02aw_tests.log
B="python bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for v in main g2 g8 static; do
  case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
  for vf in fingerprint none; do
    env $L timeout 300 $B --verify $vf > gpurun_out/r02aw_${v}_$vf.json 2> gpurun_out/r02aw_${v}_$vf.err; echo "$v $vf rc=$?"
  done
done
