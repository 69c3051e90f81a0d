# separate processes sharing one GPU (the driver's 1-GPU box): DistWorld path parity
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ae_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_multiproc_shared.py -m gpu -x -q -rA > gpurun_out/r02ae_tests.log 2>&1; echo "rc=$?"
tail -15 gpurun_out/r02ae_tests.log
