cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02n_build.log 2>&1
for n in 4 2; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=2961$n tools/stress.py --steps 1000 > gpurun_out/r02n_stress_n$n.json 2> gpurun_out/r02n_stress_n$n.err; echo "stress n$n rc=$?"
done
timeout 1200 python tools/stress.py --steps 1000 > gpurun_out/r02n_stress_n1.json 2> gpurun_out/r02n_stress_n1.err; echo "stress n1 rc=$?"
timeout 1200 python -m pytest tests/test_gpu_multiproc.py tests/test_gpu_full_size.py -q > gpurun_out/r02n_mp.log 2>&1; echo "mp rc=$?"
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02n_bench_n4.json 2> gpurun_out/r02n_bench_n4.err; echo "bench n4 rc=$?"
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02n_bench_n2.json 2> gpurun_out/r02n_bench_n2.err; echo "bench n2 rc=$?"
timeout 900 python bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > gpurun_out/r02n_ref_n2.json 2> gpurun_out/r02n_ref_n2.err; echo "ref n2 rc=$?"
tail -2 gpurun_out/r02n_mp.log
