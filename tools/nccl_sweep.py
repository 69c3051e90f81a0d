#!/usr/bin/env python
"""NCCL baseline sweep for the hpZ collectives: the same messages as
bench.py's nccl_baseline — AllGather over P of one Falcon-7B block (bf16), AllGather over the
virtual node (P' ranks), fp32 ReduceScatter(AVG) over P — timed with CUDA events (max over
ranks) under whatever NCCL_* environment the launcher sets, nccl-tests style (algbw =
output bytes / time for AG, input bytes / time for RS; busbw = algbw * (n-1)/n).

    torchrun --nproc-per-node 4 tools/nccl_sweep.py --label default
    NCCL_ALGO=NVLS torchrun ... tools/nccl_sweep.py --label nvls
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--label", default="default")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--numel", type=int, default=207_071_232)    # one Falcon-7B block, padded for P <= 8
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    P, r = dist.get_world_size(), dist.get_rank()
    node = P // 2 if P >= 2 else 1
    groups = [dist.new_group(list(range(n * node, (n + 1) * node))) for n in range(P // node)]
    g = groups[r // node]
    N = args.numel // (P * 256) * (P * 256)
    full = torch.empty(N, dtype=torch.bfloat16, device=dev)
    prim = torch.ones(N // P, dtype=torch.bfloat16, device=dev)
    sec = torch.ones(N // node, dtype=torch.bfloat16, device=dev)
    grad = torch.ones(N, dtype=torch.float32, device=dev)
    gsh = torch.empty(N // P, dtype=torch.float32, device=dev)
    ops = {"ag_world": lambda: dist.all_gather_into_tensor(full, prim),
           "ag_node": lambda: dist.all_gather_into_tensor(full, sec, group=g),
           "rs_world": lambda: dist.reduce_scatter_tensor(gsh, grad, op=dist.ReduceOp.AVG)}
    res = {}
    for name, fn in ops.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.iters):
            fn()
        b.record()
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) / args.iters], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        n_ranks = node if name == "ag_node" else P
        nbytes = N * (2 if name.startswith("ag") else 4)
        algbw = nbytes / (ms * 1e-3) / 1e9
        res[name] = {"ms": round(ms, 3), "algbw_GBps": round(algbw, 1),
                     "busbw_GBps": round(algbw * (n_ranks - 1) / n_ranks, 1)}
    if r == 0:
        env = {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}
        print(json.dumps({"label": args.label, "world": P, "node_size": node, "numel": N, "env": env,
                          "nccl": ".".join(map(str, torch.cuda.nccl.version())), "ops": res}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
