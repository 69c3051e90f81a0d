# N=1: local gathers by the TMA pipeline vs the LDG/STG kernel (per-kernel breakdown)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ad_build.log 2>&1
B="python bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-nccl --no-p2p-ceiling"
for r in 1 2; do
  timeout 300 $B > gpurun_out/r02ad_tma_$r.json 2>gpurun_out/r02ad_tma_$r.err
  for c in 1 2 4 8; do timeout 300 $B --copy-engine ldg --ctas-per-sm $c > gpurun_out/r02ad_ldg${c}_$r.json 2>gpurun_out/r02ad_ldg${c}_$r.err; done
done
