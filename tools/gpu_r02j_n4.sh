cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_multiproc.py -q > gpurun_out/r02j_mp.log 2>&1; echo "mp rc=$?"
B="python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl"
timeout 600 $B --verify none > gpurun_out/r02j_main_nov.json 2> gpurun_out/r02j_main_nov.err; echo "main nov rc=$?"
for v in main b224 g6 b224g6; do
  if [ $v = main ]; then L=""; else L="HPZ_LIB=$PWD/abtest_$v/libhpz.so"; fi
  env $L timeout 600 $B > gpurun_out/r02j_ab_$v.json 2> gpurun_out/r02j_ab_$v.err; echo "ab $v rc=$?"
done
N="python tools/nvlink_bytes.py --world 4 --node-size 2"
timeout 300 $N > gpurun_out/r02j_nvl_plain.json 2> gpurun_out/r02j_nvl_plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gather_tma|rs_tma" --launch-skip 12 --launch-count 12 --csv --log-file gpurun_out/r02j_ncu_nvl.csv $N > gpurun_out/r02j_ncu_nvl.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r02j_mp.log
