# the driver's round-end GPU tier on one GPU: full -m gpu suite + smoke + default bench
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ak_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/r02ak_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r02ak_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ak_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/r02ak_bench.json 2> gpurun_out/r02ak_bench.err; echo "bench rc=$?"
