# A/B of the RS+Adam stage geometry at N=4 as a proxy for P=8 (2 stages of 88 KiB there):
# main (2048-element chunks, 4 stages), st2 (2 stages), pn1 (1024-element chunks, 6 stages),
# pn1st8 (1024-element chunks, 8 stages)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ab_build.log 2>&1
for n in 4 2; do
  B="python bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
  for v in main st2 pn1 pn1st8 main2 st22 pn12 pn1st82; do
    case $v in main|main2) L="";; *) L="HPZ_LIB=$PWD/abtest_${v%2}/libhpz.so";; esac
    [ $v = st22 ] && L="HPZ_LIB=$PWD/abtest_st2/libhpz.so"
    env $L timeout 600 $B > gpurun_out/r02ab_n${n}_$v.json 2> gpurun_out/r02ab_n${n}_$v.err; echo "n$n $v rc=$?"
  done
done
