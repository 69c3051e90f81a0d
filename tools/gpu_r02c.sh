cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_overlap.py -q > gpurun_out/r02c_parity.log 2>&1; echo "parity rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/r02c_bench_graph.json 2> gpurun_out/r02c_bench_graph.err; echo "bench graph rc=$?"
timeout 600 $B --graph 0 > gpurun_out/r02c_bench_eager.json 2> gpurun_out/r02c_bench_eager.err; echo "bench eager rc=$?"
timeout 600 $B --verify none > gpurun_out/r02c_bench_noverify.json 2> gpurun_out/r02c_bench_noverify.err; echo "bench noverify rc=$?"
SMALL="python bench.py --model falcon7b_block --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --graph 0"
timeout 300 $SMALL > gpurun_out/r02c_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rs_tma_kernel|gather_tma_kernel" -s 3 -c 3 -o gpurun_out/r02c_prof_n1 $SMALL > gpurun_out/r02c_ncu_full.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/r02c_parity.log
