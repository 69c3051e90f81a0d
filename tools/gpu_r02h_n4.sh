# 4-GPU run: full GPU suite, bench self-launch at N=2,4 (both arms), NCCL sweep, RS geometry
# A/B at N=4, NVLink byte counters of rank 0's hot kernels (ncu, one rank).
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02h_build.log 2>&1
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/r02h_pytest.log 2>&1; echo "pytest rc=$?"
timeout 900 python bench.py --gpus 4 --steps 10 --warmup 3 > gpurun_out/r02h_bench_n4.json 2> gpurun_out/r02h_bench_n4.err; echo "bench n4 rc=$?"
timeout 900 python bench.py --impl reference --gpus 4 --steps 2 --warmup 1 > gpurun_out/r02h_ref_n4.json 2> gpurun_out/r02h_ref_n4.err; echo "ref n4 rc=$?"
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02h_bench_n2.json 2> gpurun_out/r02h_bench_n2.err; echo "bench n2 rc=$?"
for v in "default" "ring NCCL_ALGO=Ring" "nvls NCCL_ALGO=NVLS" "nvls_off NCCL_NVLS_ENABLE=0" "simple NCCL_PROTO=Simple" "ch32 NCCL_MIN_NCHANNELS=32" "ring_ch32 NCCL_ALGO=Ring NCCL_MIN_NCHANNELS=32 NCCL_PROTO=Simple"; do
  set -- $v; lab=$1; shift
  env "$@" timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29$((RANDOM % 800 + 100)) tools/nccl_sweep.py --label $lab >> gpurun_out/r02h_nccl_sweep.jsonl 2>> gpurun_out/r02h_nccl_sweep.err
done
echo "nccl sweep done"
B="python bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl"
for v in pn1 2cta st3; do
  HPZ_LIB=$PWD/abtest_$v/libhpz.so timeout 600 $B > gpurun_out/r02h_ab_$v.json 2> gpurun_out/r02h_ab_$v.err; echo "ab $v rc=$?"
done
timeout 600 $B > gpurun_out/r02h_ab_main.json 2> gpurun_out/r02h_ab_main.err; echo "ab main rc=$?"
# NVLink bytes of rank 0's hot kernels: ranks 1-3 plain, rank 0 under ncu (single-pass metrics)
export MASTER_ADDR=127.0.0.1 MASTER_PORT=29577 WORLD_SIZE=4
C="bench.py --gpus 4 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-nccl --graph 0 --verify none"
for r in 1 2 3; do RANK=$r LOCAL_RANK=$r timeout 600 python $C > /dev/null 2> gpurun_out/r02h_nvl_rank$r.err & done
RANK=0 LOCAL_RANK=0 timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"rs_tma_kernel|gather_tma_kernel" -c 9 --csv --log-file gpurun_out/r02h_ncu_nvl.csv python $C > gpurun_out/r02h_nvl_rank0.log 2>&1
echo "ncu nvl rc=$?"
wait
tail -3 gpurun_out/r02h_pytest.log
