# NVLink + DRAM bytes per launch of the hot kernels at world 4 (P'=2) and world 2 (P'=1), bench
# configuration (fingerprint, no gradient-shard store), then bench lines that carry them
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02aj_build.log 2>&1
M=gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum
for cfg in "4 2" "2 1"; do
  set -- $cfg; P=$1; Pp=$2
  N="python tools/nvlink_bytes.py --world $P --node-size $Pp"
  timeout 300 $N > gpurun_out/r02aj_plain_w$P.json 2> gpurun_out/r02aj_plain_w$P.err; echo "plain w$P rc=$?"
  timeout 900 ncu --metrics $M --clock-control none -k regex:"gather_tma|rs_tma" --launch-skip $((3*P)) --launch-count $((3*P)) --csv --log-file gpurun_out/r02aj_ncu_nvl_w$P.csv $N > gpurun_out/r02aj_ncu_w$P.log 2>&1; echo "ncu w$P rc=$?"
  python tools/nvlink_summary.py gpurun_out/r02aj_ncu_nvl_w$P.csv gpurun_out/r02aj_plain_w$P.json gpurun_out/r02aj_nvlink_bytes_w$P.json --traffic profiles/ncu_traffic.json > gpurun_out/r02aj_sum_w$P.log 2>&1; echo "sum w$P rc=$?"
done
cp profiles/ncu_traffic.json gpurun_out/r02aj_ncu_traffic.json
for n in 4 2; do
  timeout 600 python bench.py --gpus $n > gpurun_out/r02aj_bench_n$n.json 2> gpurun_out/r02aj_bench_n$n.err; echo "bench n$n rc=$?"
done
