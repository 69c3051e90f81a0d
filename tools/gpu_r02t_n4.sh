# final 4-GPU evidence: full GPU suite, stress variants (qgZ+qwZ, bf16 gradients), bench N=4/2/1 lines
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02t_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02t_pytest.log 2>&1; echo "pytest rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29631 tools/stress.py --steps 300 --qgz --qwz --verify fingerprint > gpurun_out/r02t_stress_qgz_qwz_n4.json 2> gpurun_out/r02t_stress_qgz_qwz_n4.err; echo "stress qgz rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29632 tools/stress.py --steps 300 --grad-dtype bf16 > gpurun_out/r02t_stress_bf16_n4.json 2> gpurun_out/r02t_stress_bf16_n4.err; echo "stress bf16 rc=$?"
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02t_bench_n4.json 2> gpurun_out/r02t_bench_n4.err; echo "bench n4 rc=$?"
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02t_bench_n2.json 2> gpurun_out/r02t_bench_n2.err; echo "bench n2 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02t_bench_n1.json 2> gpurun_out/r02t_bench_n1.err; echo "bench n1 rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02t_ref_n1.json 2> gpurun_out/r02t_ref_n1.err; echo "ref n1 rc=$?"
tail -3 gpurun_out/r02t_pytest.log
