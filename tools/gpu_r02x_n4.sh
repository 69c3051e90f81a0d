cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02x_build.log 2>&1
for n in 4 2; do
  B="python bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
  for v in main rot rotwl main2 rot2; do
    case $v in main|main2) L="";; rot|rot2) L="HPZ_LIB=$PWD/abtest_rot/libhpz.so";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
    env $L timeout 600 $B > gpurun_out/r02x_n${n}_$v.json 2> gpurun_out/r02x_n${n}_$v.err; echo "n$n $v rc=$?"
  done
done
