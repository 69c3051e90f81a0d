# the driver's default N=8 bench command (full falcon7b, e2e on) with 8 ranks on 4 GPUs
# (2 time-sliced ranks per GPU = twice the real per-GPU footprint): functional + memory check
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ag_build.log 2>&1
( while sleep 20; do nvidia-smi --query-gpu=index,memory.used --format=csv,noheader; done ) > gpurun_out/r02ag_mem.log 2>&1 &
M=$!
timeout 1200 python bench.py --gpus 8 --share-gpus --steps 2 --warmup 3 > gpurun_out/r02ag_bench8.json 2> gpurun_out/r02ag_bench8.err; echo "bench rc=$?"
timeout 900 python bench.py --gpus 8 --share-gpus --node-size 2 --steps 2 --warmup 3 --no-e2e > gpurun_out/r02ag_bench8_4x2.json 2> gpurun_out/r02ag_bench8_4x2.err; echo "bench 4x2 rc=$?"
kill $M
sort -t, -k2 -n gpurun_out/r02ag_mem.log | tail -4
