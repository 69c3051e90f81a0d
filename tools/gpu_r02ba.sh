# bench after the byte-accounting refactor: N=1 line and the N>1 path (2 ranks sharing the GPU)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02ba_build.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02ba_n1.json 2> gpurun_out/r02ba_n1.err; echo "n1 rc=$?"
timeout 600 python bench.py --gpus 2 --share-gpus --model falcon7b_block --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02ba_n2s.json 2> gpurun_out/r02ba_n2s.err; echo "n2s rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r02ba_ref.json 2> gpurun_out/r02ba_ref.err; echo "ref rc=$?"
