cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02r_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "concurrent or missing_peer" > gpurun_out/r02r_conc.log 2>&1; echo "conc rc=$?"
tail -3 gpurun_out/r02r_conc.log
