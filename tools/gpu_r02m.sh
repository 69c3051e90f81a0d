cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02m_build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02m_pytest.log 2>&1; echo "pytest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02m_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02m_bench_n1.json 2> gpurun_out/r02m_bench_n1.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --verify none --no-cpu-baseline --no-e2e > gpurun_out/r02m_bench_n1_nov.json 2> gpurun_out/r02m_bench_n1_nov.err; echo "bench nov rc=$?"
tail -3 gpurun_out/r02m_pytest.log
