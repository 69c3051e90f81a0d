cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02al_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_full_size.py -m gpu -q -rA -k sharing > gpurun_out/r02al_tests.log 2>&1; echo "rc=$?"; tail -4 gpurun_out/r02al_tests.log
