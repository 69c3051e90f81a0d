#!/usr/bin/env python
"""Config C5: the stale-weight stress — Llama-2-70B layer-shaped flat buffers streamed per
layer for many steps, fixed ordering (the paper's fix) vs the stock ZeRO++ ordering.

    python tools/stress.py --steps 1000                     # N=1
    torchrun --nproc-per-node N tools/stress.py --steps 1000

Every backward gather is checked element by element against the owners' primaries
(HPZ_VERIFY_EXACT, a7) and by the fwd/bwd fingerprint; rank 0 prints one JSON line with
the mismatch counts of the fixed run (must be 0) and of the stock run (must be > 0:
Table 1's "x").  Gradients are regenerated on the device every step
(synthetic, seeded), so the gradient-slot edges E5/E6 are exercised too.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run(order, args, world, rank, local, node_size, numels):
    import torch
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import DistWorld, EmulatedWorld, sum_over_ranks
    from synth import inputs as S
    # the stock race needs a secondary of its own (at P' == P it is aliased to the primary)
    kw = dict(n_grad_slots=2, timeout_s=60.0, qgz=args.qgz, qwz=args.qwz, grad_dtype=args.grad_dtype,
              alias_secondary=order != "stock")
    if world > 1:
        W = DistWorld(numels, node_size, device=local, **kw)
    else:
        W = EmulatedWorld(numels, 1, 1, device=local, **kw)
    rc = W.ranks[0]
    ctx = rc.ctx
    s = torch.cuda.current_stream()
    H.hpz_set_order(ctx, order, stock_delay_us=args.stock_delay_us if order == "stock" else 0,
                    stock_poison=order == "stock")
    # EXACT compares against raw primaries: not meaningful with qwZ (dequantized gathers)
    H.hpz_set_verify(ctx, "fingerprint" if (args.qwz or args.verify == "fingerprint") else "exact")
    L = len(numels)
    for i in range(L):
        H.hpz_synth_master(ctx, i, S.stream_key(S.SEED_PARAMS, i, 0, 0), S.PARAM_SCALE, s)
    nmax = max(x.numel_pad for x in rc.infos)
    # one full buffer per layer for the stock run: the side-stream copy reads it late
    fwd = [torch.empty(nmax, dtype=torch.bfloat16, device="cuda") for _ in range(L if order == "stock" else 1)]
    bwd = torch.empty(nmax, dtype=torch.bfloat16, device="cuda")
    adam = H.make_adam()
    torch.cuda.synchronize()
    t0 = time.time()
    steps = args.steps if order == "fixed" else args.stock_steps
    for t in range(steps):
        for i in range(L):
            H.hpz_fwd_gather(ctx, i, fwd[i % len(fwd)].data_ptr(), s)
        for i in reversed(range(L)):
            H.hpz_bwd_gather(ctx, i, bwd.data_ptr(), s)
            H.hpz_synth_grads(ctx, i, S.stream_key(S.SEED_GRADS, i, t, rank), S.GRAD_SCALE, 0, s)
            H.hpz_reduce_scatter_adam(ctx, i, adam, s)
    torch.cuda.synchronize()
    secs = time.time() - t0
    c = H.hpz_counters(ctx)
    tot = sum_over_ranks([c["mismatches"], c["nan_reads"], c["fp_mismatches"], c["fp_checked"], c["timeouts"],
                          c["fp_fwd_mismatches"], c["fp_fwd_checked"]], device=torch.device("cuda", local))
    W.close()
    return {"order": order, "steps": steps, "wall_s": round(secs, 1), "mismatched_elements": int(tot[0]),
            "nan_reads": int(tot[1]), "fingerprint_mismatched_layers": int(tot[2]),
            "layer_gathers_checked": int(tot[3]), "timeouts": int(tot[4]),
            "fwd_vs_owner_fingerprint_mismatched_layers": int(tot[5]), "fwd_layer_gathers_checked": int(tot[6])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--stock-steps", type=int, default=3)
    ap.add_argument("--stock-delay-us", type=int, default=20000)
    ap.add_argument("--model", default="llama2_70b_layers")
    ap.add_argument("--qgz", action="store_true")
    ap.add_argument("--qwz", action="store_true")
    ap.add_argument("--grad-dtype", default="f32")
    ap.add_argument("--verify", default="exact", choices=["exact", "fingerprint"])
    ap.add_argument("--node-size", type=int, default=0, help="P' (default N/2)")
    ap.add_argument("--share-gpus", action="store_true",
                    help="rank r on GPU r %% #GPUs (e.g. the 8-rank topologies on a 4-GPU box; gloo control plane)")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.share_gpus:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if args.share_gpus:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    node_size = args.node_size or (world // 2 if world >= 2 else 1)
    from paper_2407_01614_b200 import shapes
    numels = shapes.numels(args.model)
    res = [run("fixed", args, world, rank, local, node_size, numels)]
    if args.stock_steps > 0:
        res.append(run("stock", args, world, rank, local, node_size, numels))
    if rank == 0:
        out = {"config": f"C5 stress: {args.model} ({len(numels)} x {numels[0]} elements), P={world}, P'={node_size}"
                         + (f", {world} processes sharing {torch.cuda.device_count()} GPU(s) (time-sliced)"
                            if args.share_gpus else ""),
               "options": {"qgz": args.qgz, "qwz": args.qwz, "grad_dtype": args.grad_dtype},
               "runs": res,
               "pass": res[0]["mismatched_elements"] == 0 and res[0]["fingerprint_mismatched_layers"] == 0
               and res[0]["fwd_vs_owner_fingerprint_mismatched_layers"] == 0 and res[0]["timeouts"] == 0
               and (len(res) < 2 or res[1]["mismatched_elements"] > 0 or res[1]["fingerprint_mismatched_layers"] > 0)}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
