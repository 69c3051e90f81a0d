# model sweep (BASELINE configs C2-C5 shapes) at N = 1, 2, 4 + C3's node-size sweep + the
# f3 Table-2 analog with the corrected ORDER_PAPER (no caller-stream stall after the copy)
cd $GRAFT_REPO_ROOT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02p_build.log 2>&1
run() { m=$1; n=$2; tag=$3; shift 3
  out=gpurun_out/r02p_sweep_${m}_n${n}${tag}.json
  timeout 900 python bench.py --gpus $n --model $m --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-p2p-ceiling "$@" > $out.log 2>&1
  rc=$?; grep '^{' $out.log | tail -1 > $out; echo "$m n=$n $tag rc=$rc"
}
for n in 1 2 4; do
  run falcon7b $n ""
  run llama2_7b $n ""
  run falcon40b_block $n ""
  run llama2_70b_layers $n ""
done
run llama2_13b 2 "_p2" --grad-slots 2
run llama2_13b 2 "_p1" --grad-slots 2 --node-size 1
run llama2_13b 4 "_p2" --grad-slots 2
run llama2_13b 4 "_p4" --grad-slots 2 --node-size 4
run falcon40b_block 4 "_p4" --node-size 4
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 --master-port=2978$n \
    tools/train_overlap.py --model transformer --h 4096 --heads 32 --ffn 11008 --seq 1024 --tokens 1024 --qgz \
    --configs off:1,fixed:1,paper:1,stock:1 > gpurun_out/r02p_f3_qgz_n$n.log 2>&1; echo "f3 n$n rc=$?"
  grep '^{' gpurun_out/r02p_f3_qgz_n$n.log | tail -1 > gpurun_out/r02p_f3_qgz_n$n.json
done
