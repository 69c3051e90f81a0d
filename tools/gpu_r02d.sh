cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02d_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_stock_schedule.py tests/test_gpu_parity.py -q -x -k "stock or fingerprint or captured" > gpurun_out/r02d_new.log 2>&1; echo "new rc=$?"
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $B > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; echo "bench rc=$?"
timeout 600 $B --verify none > gpurun_out/r02d_bench_nov.json 2> gpurun_out/r02d_bench_nov.err; echo "bench nov rc=$?"
HPZ_LIB=$PWD/abtest_p1x2/libhpz.so timeout 600 $B > gpurun_out/r02d_bench_p1x2.json 2> gpurun_out/r02d_bench_p1x2.err; echo "bench p1x2 rc=$?"
HPZ_LIB=$PWD/abtest_p1x2/libhpz.so timeout 600 $B --verify none > gpurun_out/r02d_bench_p1x2_nov.json 2> gpurun_out/r02d_bench_p1x2_nov.err; echo "bench p1x2 nov rc=$?"
tail -3 gpurun_out/r02d_new.log
