cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02i_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_wide.py -q -x -k "fingerprint or captured or special or ring or fused or qwz" > gpurun_out/r02i_tests.log 2>&1; echo "tests rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/r02i_bench.json 2> gpurun_out/r02i_bench.err; echo "bench rc=$?"
timeout 600 $B --verify none > gpurun_out/r02i_bench_nov.json 2> gpurun_out/r02i_bench_nov.err; echo "bench nov rc=$?"
tail -3 gpurun_out/r02i_tests.log
