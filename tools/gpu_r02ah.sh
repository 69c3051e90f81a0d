# N=1 local-gather geometry A/B (chunk x stages), plus verify=none to price the fingerprint warps
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ah_build.log 2>&1
B="python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
for r in 1 2; do
  for v in main lc32s6 lc16s12 lc8s24 lc64s3 vnone; do
    case $v in main) L=""; X="";; vnone) L=""; X="--verify none";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so"; X="";; esac
    env $L timeout 300 $B $X > gpurun_out/r02ah_${v}_$r.json 2> gpurun_out/r02ah_${v}_$r.err; echo "$v $r rc=$?"
  done
done
