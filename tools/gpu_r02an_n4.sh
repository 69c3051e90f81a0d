# remote gather stage ring A/B at N=4 and N=2: 32 KiB x 4 (main) vs x3, x2, 64 KiB x 2
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02an_build.log 2>&1
for n in 4 2; do
  B="python bench.py --gpus $n --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
  for r in 1 2; do
    for v in main g3 g2 g64x2; do
      case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
      env $L timeout 600 $B > gpurun_out/r02an_n${n}_${v}_$r.json 2> gpurun_out/r02an_n${n}_${v}_$r.err; echo "n$n $v $r rc=$?"
    done
  done
done
