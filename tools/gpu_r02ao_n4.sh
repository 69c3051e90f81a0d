# adopted geometry (remote gathers 32 KiB x 3, RS <= 2 stages at P >= 4) vs the previous
# default (prev) and the gather change alone (g3only), N=4 and N=2, interleaved; then the
# GPU parity suites with the new default
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ao_build.log 2>&1
for n in 4 2; do
  B="python bench.py --gpus $n --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
  for r in 1 2; do
    for v in main prev g3only; do
      case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
      env $L timeout 600 $B > gpurun_out/r02ao_n${n}_${v}_$r.json 2> gpurun_out/r02ao_n${n}_${v}_$r.err; echo "n$n $v $r rc=$?"
    done
  done
done
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02ao_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02ao_tests.log
