# gather chunk order: dynamic (main), dynamic with the counter read one ahead (dyn2), static; with
# and without fingerprint warps
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02at_build.log 2>&1
HPZ_LIB=$PWD/abtest_dyn2/libhpz.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "fixed or alias or replay" > gpurun_out/r02at_tests_dyn2.log 2>&1; echo "tests dyn2 rc=$?"; tail -1 gpurun_out/r02at_tests_dyn2.log
B="python bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for v in main dyn2 static; do
  case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
  for vf in fingerprint none; do
    env $L timeout 300 $B --verify $vf > gpurun_out/r02at_${v}_$vf.json 2> gpurun_out/r02at_${v}_$vf.err; echo "$v $vf rc=$?"
  done
done
