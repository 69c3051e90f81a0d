cd $GRAFT_REPO_ROOT
for c in 1 2 4; do timeout 120 ./tools/mc_probe 4 512 $c; done > gpurun_out/r02w_mc.log 2>&1; echo "mc rc=$?"
timeout 120 ./tools/p2p_probe 4 pull_tma 512 1 32768 >> gpurun_out/r02w_mc.log 2>&1
timeout 120 ./tools/p2p_probe 4 push_tma 512 1 32768 >> gpurun_out/r02w_mc.log 2>&1
timeout 120 ./tools/mc_probe 2 512 4 >> gpurun_out/r02w_mc.log 2>&1
timeout 120 ./tools/p2p_probe 2 pull_tma 512 1 32768 >> gpurun_out/r02w_mc.log 2>&1
cat gpurun_out/r02w_mc.log
