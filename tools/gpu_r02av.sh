# ncu --set full of the N=1 gathers: dynamic chunk order (main) vs static, fingerprint on
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02av_build.log 2>&1
N="python tools/nvlink_bytes.py --world 1 --node-size 1"
timeout 300 $N > gpurun_out/r02av_plain.log 2>&1; echo "plain rc=$?"
for v in main static; do
  case $v in main) L="";; *) L="HPZ_LIB=$PWD/abtest_$v/libhpz.so";; esac
  env $L timeout 900 ncu --set full --import-source on --clock-control none -k regex:"gather_tma" --launch-skip 2 --launch-count 1 -o gpurun_out/r02av_$v -f $N > gpurun_out/r02av_ncu_$v.log 2>&1; echo "ncu $v rc=$?"
done
