# final 4-GPU evidence: full GPU suite, stress variants (qgZ+qwZ, bf16 gradients), bench N=4/2/1 lines
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02z_build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r02z_pytest.log 2>&1; echo "pytest rc=$?"


timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02z_bench_n4.json 2> gpurun_out/r02z_bench_n4.err; echo "bench n4 rc=$?"
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02z_bench_n2.json 2> gpurun_out/r02z_bench_n2.err; echo "bench n2 rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02z_bench_n1.json 2> gpurun_out/r02z_bench_n1.err; echo "bench n1 rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02z_ref_n1.json 2> gpurun_out/r02z_ref_n1.err; echo "ref n1 rc=$?"
tail -3 gpurun_out/r02z_pytest.log
