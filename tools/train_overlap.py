#!/usr/bin/env python
"""f3 experiment: a Table 2 / Table 1 analog on B200.

Trains the toy L-layer ReLU network of paper_2407_01614_b200.overlap with real bf16 GEMMs
(cuBLAS via torch) on the compute stream and libhpz's gathers / RS+Adam on a comm stream
(Alg. 1 PrefetchAllGather, depth 1), for orders off (no hpZ), stock (the race) and fixed
(the paper's fix).  Reports tokens/s for the whole job and per virtual node (the paper's
metric is tokens/s/node) and the loss trajectory (Table 1: stock -> NaN).

    python tools/train_overlap.py                       # N=1
    torchrun --nproc-per-node N tools/train_overlap.py  # P=N, P'=N/2
"""
import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(order, depth, args, world, rank, local, node_size):
    import torch
    import torch.distributed as dist
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.overlap import PrefetchTrainer
    from paper_2407_01614_b200.world import DistWorld, EmulatedWorld, max_over_ranks
    from synth import inputs as S
    from paper_2407_01614_b200.overlap import block_numel
    per_layer = args.h * args.h if args.model == "mlp" else block_numel(args.h, args.ffn)
    numels = [per_layer] * args.layers
    # qgZ (the paper's Table 2 runs every hpZ variant with qgZ) quantizes fp32 gradients
    kw = dict(n_grad_slots=len(numels), timeout_s=60.0, grad_dtype="f32" if args.qgz else "bf16", qgz=args.qgz,
              alias_secondary=order not in ("stock", "paper"))   # the stock / paper copies need a secondary
    W = DistWorld(numels, node_size, device=local, **kw) if world > 1 else EmulatedWorld(numels, 1, 1, device=local, **kw)
    rc = W.ranks[0]
    H.hpz_set_order(rc.ctx, order, stock_delay_us=args.stock_delay_us if order == "stock" else 0,
                    stock_poison=order == "stock")
    H.hpz_set_verify(rc.ctx, "fingerprint")
    if args.max_ctas:
        H.hpz_set_option(rc.ctx, "max_ctas", args.max_ctas)
    s = torch.cuda.current_stream()
    for i in range(args.layers):
        H.hpz_synth_master(rc.ctx, i, S.stream_key(S.SEED_PARAMS, i, 0, 0), args.init_scale, s)
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    shape = (args.tokens, args.h) if args.model == "mlp" else (args.tokens // args.seq, args.seq, args.h)
    x = (torch.randn(*shape, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    y = (x.float() * 0.05).to(torch.bfloat16)     # learnable target: a scaled copy of the input
    tr = PrefetchTrainer(rc, args.h, args.layers, args.tokens, depth=depth, lr=args.lr, model=args.model,
                         ffn=args.ffn, n_heads=args.heads, grad_dtype="f32" if args.qgz else "bf16")
    torch.cuda.synchronize()
    losses = []
    for _ in range(args.warmup):
        losses.append(tr.step(x, y))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(tr.comp)
    for _ in range(args.steps):
        losses.append(tr.step(x, y))
    tr.comp.wait_stream(tr.comm)
    b.record(tr.comp)
    torch.cuda.synchronize()
    ms = max_over_ranks([a.elapsed_time(b) / args.steps], device=torch.device("cuda", local))[0]
    lv = [float(l) for l in losses]
    c = H.hpz_counters(rc.ctx)
    W.close()
    tokens = world * args.tokens
    return {"order": order, "prefetch_depth": depth, "ms_per_step": round(ms, 3),
            "tokens_per_s": round(tokens / (ms * 1e-3), 1),
            "tokens_per_s_per_node": round(tokens / (ms * 1e-3) / max(1, world // node_size), 1),
            "loss_first": lv[0], "loss_last": lv[-1], "losses": [round(v, 6) for v in lv],
            "nan_loss": any(not math.isfinite(v) for v in lv),
            "fingerprint_mismatched_layers": c["fp_mismatches"], "timeouts": c["timeouts"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="mlp", choices=["mlp", "transformer"])
    ap.add_argument("--qgz", action="store_true", help="INT4 gradient all-to-all (fp32 gradient slots)")
    ap.add_argument("--ffn", type=int, default=5632, help="transformer MLP width")
    ap.add_argument("--heads", type=int, default=16)
    ap.add_argument("--seq", type=int, default=1024, help="transformer sequence length (tokens = batch x seq)")
    ap.add_argument("--h", type=int, default=4096)
    ap.add_argument("--layers", type=int, default=8)
    ap.add_argument("--tokens", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--max-ctas", type=int, default=32)
    ap.add_argument("--stock-delay-us", type=int, default=2000)
    ap.add_argument("--configs", default="off:1,fixed:0,fixed:1,paper:1,stock:1")
    ap.add_argument("--init-scale", type=float, default=2.0 ** -5, help="uniform init bound (~sqrt(3/h))")
    ap.add_argument("--lr", type=float, default=1e-5)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    node_size = world // 2 if world >= 2 else 1
    res = []
    for cfg in args.configs.split(","):
        order, depth = cfg.split(":")
        res.append(run(order, int(depth), args, world, rank, local, node_size))
    if rank == 0:
        by = {f"{r['order']}:{r['prefetch_depth']}": r for r in res}
        what = ("toy ReLU net" if args.model == "mlp" else
                f"pre-norm transformer blocks (h {args.h}, {args.heads} heads, GELU MLP {args.ffn}, seq {args.seq}, "
                f"activation checkpointing)")
        out = {"experiment": f"f3 Table 1/2 analog: {what}, bf16 compute + hpZ collectives on a comm stream",
               "model": args.model, "qgz": args.qgz, "world": world,
               "node_size": node_size, "h": args.h,
               "layers": args.layers,
               "tokens_per_rank": args.tokens, "max_ctas": args.max_ctas, "runs": res}
        if "fixed:1" in by and "off:1" in by:
            out["fixed_vs_off_loss_identical"] = by["fixed:1"]["loss_last"] == by["off:1"]["loss_last"]
        if "fixed:1" in by and "fixed:0" in by:
            out["prefetch_speedup"] = round(by["fixed:0"]["ms_per_step"] / by["fixed:1"]["ms_per_step"], 3)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
