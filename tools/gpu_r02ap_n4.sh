# final bench lines on the final code (remote gathers 32 KiB x 3, RS cap, probe ceiling over depths)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ap_build.log 2>&1
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02ap_bench_n4.json 2> gpurun_out/r02ap_bench_n4.err; echo "bench n4 rc=$?"
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02ap_bench_n2.json 2> gpurun_out/r02ap_bench_n2.err; echo "bench n2 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02ap_bench_n1.json 2> gpurun_out/r02ap_bench_n1.err; echo "bench n1 rc=$?"
timeout 900 python bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > gpurun_out/r02ap_ref_n4.json 2> gpurun_out/r02ap_ref_n4.err; echo "ref n4 rc=$?"
for g in 2 4; do for d in 2 3 4; do timeout 120 ./tools/p2p_probe $g pull_tma 512 1 32768 0 50 $d; done; done > gpurun_out/r02ap_probe_depths.log 2>&1
cat gpurun_out/r02ap_probe_depths.log | grep GB/s
