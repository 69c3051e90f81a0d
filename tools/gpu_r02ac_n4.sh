# A/B of the RS+Adam stage count at N=4 (P=4: 56 KiB stages; main = 4 stages), 3 interleaved reps
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ac_build.log 2>&1
B="python bench.py --gpus 4 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
for r in 1 2 3; do
  for v in main st2 st3 pn1st8; do
    case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
    env $L timeout 600 $B > gpurun_out/r02ac_n4_${v}_$r.json 2> gpurun_out/r02ac_n4_${v}_$r.err; echo "$v $r rc=$?"
  done
done
