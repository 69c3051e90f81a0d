# final code on 4 GPUs: the whole GPU suite + bench N=4 line
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02az_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02az_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02az_tests.log
timeout 900 python bench.py --gpus 4 > gpurun_out/r02az_bench_n4.json 2> gpurun_out/r02az_bench_n4.err; echo "bench n4 rc=$?"
