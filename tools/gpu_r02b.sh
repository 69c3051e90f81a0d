cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "fingerprint or captured or device_epoch or aliased" > gpurun_out/r02b_new.log 2>&1; echo "new rc=$?"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02b_pytest.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02b_bench_n1.json 2> gpurun_out/r02b_bench_n1.err; echo "bench rc=$?"
tail -3 gpurun_out/r02b_new.log gpurun_out/r02b_pytest.log
