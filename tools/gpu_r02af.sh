# 8-rank bench path and multi-process parity with ranks sharing the box's GPU(s)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02af_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multiproc_shared.py -m gpu -x -q -rA > gpurun_out/r02af_tests.log 2>&1; echo "rc=$?"
tail -12 gpurun_out/r02af_tests.log
timeout 600 python bench.py --gpus 8 --share-gpus --model falcon7b_block --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02af_bench8.json 2> gpurun_out/r02af_bench8.err; echo "bench rc=$?"
