cd $GRAFT_REPO_ROOT
timeout 300 ./tools/copy_probe > gpurun_out/r02ar_copy_probe.log 2>&1; echo "rc=$?"; cat gpurun_out/r02ar_copy_probe.log
