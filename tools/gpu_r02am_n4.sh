# C5 stress at the north_star's 8-rank topologies (2x4, 4x2) with 8 processes on 4 GPUs
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02am_build.log 2>&1
for Pp in 4 2; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=8 --master-addr 127.0.0.1 --master-port=$((29500+Pp)) \
    tools/stress.py --steps 1000 --share-gpus --node-size $Pp > gpurun_out/r02am_stress8_pp$Pp.json 2> gpurun_out/r02am_stress8_pp$Pp.err
  echo "stress P'=$Pp rc=$?"; tail -1 gpurun_out/r02am_stress8_pp$Pp.json | cut -c1-600
done
