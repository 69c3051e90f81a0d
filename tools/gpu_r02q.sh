cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02q_build.log 2>&1
timeout 900 python tools/diag_concurrent.py > gpurun_out/r02q_diag.log 2>&1; echo "diag rc=$?"
tail -60 gpurun_out/r02q_diag.log
