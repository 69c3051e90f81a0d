# final code, another 4-GPU box: N=4 and N=2 lines (box-to-box spread)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02bc_build.log 2>&1
timeout 900 python bench.py --gpus 4 > gpurun_out/r02bc_bench_n4.json 2> gpurun_out/r02bc_bench_n4.err; echo "bench n4 rc=$?"
timeout 900 python bench.py --gpus 2 > gpurun_out/r02bc_bench_n2.json 2> gpurun_out/r02bc_bench_n2.err; echo "bench n2 rc=$?"
