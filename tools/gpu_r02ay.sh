# N=1: wide local gathers with one flag-acquire kernel before each (main), with per-CTA acquires
# (noprew), 64 KiB CTAs (big), the previous persistent TMA gathers (old)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ay_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -m gpu -x -q > gpurun_out/r02ay_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02ay_tests.log
B="python bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
for r in 1 2; do
for v in main noprew big old; do
  case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
  env $L timeout 300 $B > gpurun_out/r02ay_${v}_$r.json 2> gpurun_out/r02ay_${v}_$r.err; echo "$v $r rc=$?"
done
done
