#!/usr/bin/env python
"""NVLink byte counters of the hot kernels, per launch ("no NVLink counter confirms
any of these GB/s figures").

`ncu` must never wrap a multi-rank command (B200_PROFILING.md), so this drives P GPUs from ONE
process: one libhpz context per GPU (hpz_init(..., device=r)), every arena allocated on its own
GPU and bound into every context through peer access (hpz_bind), every rank's calls issued on
its own device's stream in SPMD phase order (all ranks' forward gathers of a layer, then all
backward gathers, gradients, E5, fused RS+Adam) — so each flag a kernel waits for was released
by a kernel issued before it, and `ncu`'s kernel serialization cannot deadlock.  Under `ncu
--metrics nvlrx__bytes.sum,nvltx__bytes.sum,...` each profiled kernel runs alone, so the
device's NVLink counters during its window are its own traffic.

    ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,\\
        dram__bytes_write.sum -k regex:"gather_tma|rs_tma" --launch-skip 6 --launch-count 6 --csv \\
        python tools/nvlink_bytes.py --world 2 --node-size 1
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def enable_peer_access(n):
    rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if rt is None:
        rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
    for d in range(n):
        rt.cudaSetDevice(d)
        for q in range(n):
            if q != d:
                e = rt.cudaDeviceEnablePeerAccess(q, 0)
                if e not in (0, 704):          # 704 = already enabled
                    raise RuntimeError(f"cudaDeviceEnablePeerAccess({d}->{q}) = {e}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--node-size", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--model", default="falcon7b_block")
    ap.add_argument("--verify", default="fingerprint", choices=["none", "fingerprint"],
                    help="the bench's default is fingerprint")
    args = ap.parse_args()
    import torch
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200 import shapes
    from synth import inputs as S
    P, Pp = args.world, args.node_size
    numels = shapes.numels(args.model)
    for d in range(P):
        torch.cuda.set_device(d)
        torch.cuda.synchronize()
    enable_peer_access(P)
    ctxs = []
    for r in range(P):
        ctx = H.hpz_init(P, Pp, r, r)
        H.hpz_register_flat_params(ctx, numels)
        H.hpz_arena_alloc(ctx)
        H.hpz_set_verify(ctx, args.verify)
        H.hpz_set_option(ctx, "store_grad_shard", 0)   # the bench's fused RS+Adam stores no gradient shard
        ctxs.append(ctx)
    ptrs = [H.hpz_arena_ptr(c, r) for r, c in enumerate(ctxs)]
    for r, c in enumerate(ctxs):
        torch.cuda.set_device(r)
        H.hpz_bind(c, ptrs)
    infos = [H.hpz_layer_info(ctxs[0], i) for i in range(len(numels))]
    streams = [torch.cuda.Stream(device=r) for r in range(P)]
    bufs = [torch.empty(max(x.numel_pad for x in infos), dtype=torch.bfloat16, device=f"cuda:{r}") for r in range(P)]
    L = len(numels)
    adam = H.make_adam()

    def each(fn):
        for r in range(P):
            with torch.cuda.device(r):
                fn(r, ctxs[r], streams[r])

    each(lambda r, c, s: [H.hpz_synth_master(c, i, S.stream_key(S.SEED_PARAMS, i, 0, 0), S.PARAM_SCALE, s)
                          for i in range(L)])
    for t in range(args.steps):
        for i in range(L):
            each(lambda r, c, s: H.hpz_fwd_gather(c, i, bufs[r].data_ptr(), s))
        for i in reversed(range(L)):
            each(lambda r, c, s: H.hpz_bwd_gather(c, i, bufs[r].data_ptr(), s))
            each(lambda r, c, s: H.hpz_synth_grads(c, i, S.stream_key(S.SEED_GRADS, i, t, r), S.GRAD_SCALE, 0, s))
            each(lambda r, c, s: H.hpz_grads_ready(c, i, s))
            each(lambda r, c, s: H.hpz_reduce_scatter_adam(c, i, adam, s))
    for r in range(P):
        torch.cuda.synchronize(r)
    cnt = [H.hpz_counters(c) for c in ctxs]
    e = 2
    # this GPU's own DRAM bytes per launch (its peers idle under ncu): own shard / secondary
    # read, full buffer (+ secondary) written; RS+Adam: own gradient slice read, master/m/v
    # read + written, bf16 primary written
    hbm = {"fwd_gather": [x.shard * e + x.numel_pad * e + (x.sec_shard * e if Pp < P else 0) for x in infos],
           "bwd_gather": [x.sec_shard * e + x.numel_pad * e for x in infos],
           "reduce_scatter+adam": [x.shard * (4 + 12 + 12 + e) for x in infos]}
    alg = {"fwd_gather": [x.numel_pad * e * (P - 1) // P for x in infos],
           "bwd_gather": [x.numel_pad * e * (Pp - 1) // Pp for x in infos],
           "reduce_scatter+adam": [x.numel_pad * 4 * (P - 1) // P for x in infos]}
    print(json.dumps({"world": P, "node_size": Pp, "model": args.model, "numel_pad": [x.numel_pad for x in infos],
                      "nvlink_ingress_alg_bytes_per_launch": alg, "local_hbm_alg_bytes_per_launch": hbm,
                      "timeouts": sum(x["timeouts"] for x in cnt)}), flush=True)
    for c in ctxs:
        H.hpz_finalize(c)


if __name__ == "__main__":
    main()
