cd $GRAFT_REPO_ROOT
timeout 300 python tools/copy_ceiling.py > gpurun_out/r02aq_copy.json 2> gpurun_out/r02aq_copy.err; echo "rc=$?"; cat gpurun_out/r02aq_copy.json
