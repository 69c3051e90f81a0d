"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(TMA engine, fused RS+Adam, resident synthetic gradients, fingerprint verification):
Falcon-7B-shaped flat buffers, a few steps, then sampled elements compared with the
oracle computed one element at a time (oracle.sampled_trajectory).

    python tests/full_size_worker.py                      # N=1 (P=1)
    torchrun --nproc-per-node N tests/full_size_worker.py # P=N, P'=N/2
    HPZ_SHARE_GPUS=1 HPZ_FULL_MODEL=falcon7b_block torchrun --nproc-per-node 8 ...  # 8 ranks, any #GPUs
Prints FULL_SIZE_OK on success (rank 0)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    import torch.distributed as dist
    from oracle import hpz_oracle as O
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200 import shapes
    from paper_2407_01614_b200.world import DistWorld, EmulatedWorld, buffer_view, sum_over_ranks
    from synth import inputs as S
    model = os.environ.get("HPZ_FULL_MODEL", "falcon7b")
    steps = int(os.environ.get("HPZ_FULL_STEPS", "3"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    share = os.environ.get("HPZ_SHARE_GPUS") == "1"   # rank r on GPU r % #GPUs (time-sliced processes)
    if share:
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")             # NCCL refuses two ranks on one device
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    node = world // 2 if world >= 2 else 1
    numels = shapes.numels(model)
    L = len(numels)
    W = DistWorld(numels, node, n_grad_slots=L, device=local) if world > 1 else \
        EmulatedWorld(numels, 1, 1, n_grad_slots=L, device=local)
    rc = W.ranks[0]
    ctx = rc.ctx
    H.hpz_set_verify(ctx, "fingerprint")
    H.hpz_set_option(ctx, "store_grad_shard", 0)
    s = torch.cuda.current_stream()
    for i in range(L):
        H.hpz_synth_master(ctx, i, S.stream_key(S.SEED_PARAMS, i, 0, 0), S.PARAM_SCALE, s)
        H.hpz_synth_grads(ctx, i, S.stream_key(S.SEED_GRADS, i, 0, rank), S.GRAD_SCALE, 0, s)
    nmax = max(x.numel_pad for x in rc.infos)
    fwd = torch.empty(nmax, dtype=torch.bfloat16, device="cuda")
    bwd = torch.empty(nmax, dtype=torch.bfloat16, device="cuda")
    adam = H.make_adam()
    check_layers = sorted({i for i in (0, 1, L - 1) if i < L})
    rng = np.random.default_rng(11)
    samples = {i: np.unique(np.concatenate([rng.integers(0, numels[i], 3000),
                                            [0, numels[i] - 1, rc.infos[i].numel_pad - 1]]))
               for i in check_layers}
    fails = []
    for t in range(steps):
        for i in range(L):
            H.hpz_fwd_gather(ctx, i, fwd.data_ptr(), s)
            if i in check_layers:                       # W_t at sampled positions, every rank
                got = fwd[torch.from_numpy(samples[i]).cuda()].view(torch.int16).cpu().numpy().view(np.uint16)
                _, _, _, p = O.sampled_trajectory(i, numels[i], world, samples[i], t, O.AdamHyper(), fixed_grads=True)
                if not np.array_equal(got, p):
                    fails.append(f"fwd t={t} layer={i}")
        for i in reversed(range(L)):
            H.hpz_bwd_gather(ctx, i, bwd.data_ptr(), s)
            if i in check_layers:
                got = bwd[torch.from_numpy(samples[i]).cuda()].view(torch.int16).cpu().numpy().view(np.uint16)
                _, _, _, p = O.sampled_trajectory(i, numels[i], world, samples[i], t, O.AdamHyper(), fixed_grads=True)
                if not np.array_equal(got, p):
                    fails.append(f"bwd t={t} layer={i}")
            H.hpz_reduce_scatter_adam(ctx, i, adam, s)
    torch.cuda.synchronize()
    # optimizer state of my shard at sampled positions (global index -> my shard)
    for i in check_layers:
        info = rc.infos[i]
        lo, hi = rank * info.shard, (rank + 1) * info.shard
        mine = samples[i][(samples[i] >= lo) & (samples[i] < hi)]
        if mine.size == 0:
            continue
        w, m, v, p = O.sampled_trajectory(i, numels[i], world, mine, steps, O.AdamHyper(), fixed_grads=True)
        loc = torch.from_numpy(mine - lo).cuda()
        for kind, ref in (("master", w), ("m", m), ("v", v)):
            got = buffer_view(rc, i, kind, "f32")[loc].cpu().numpy()
            if not np.array_equal(got.view(np.uint32), ref.view(np.uint32)):
                fails.append(f"{kind} layer={i}")
        gp = buffer_view(rc, i, "primary", "bf16")[loc].view(torch.int16).cpu().numpy().view(np.uint16)
        if not np.array_equal(gp, p):
            fails.append(f"primary layer={i}")
    c = H.hpz_counters(ctx)
    bad = sum_over_ranks([len(fails), c["fp_mismatches"], c["timeouts"]], device=torch.device("cuda", local))
    W.close()
    if rank == 0:
        print("failures:", fails, "fp_mismatches", bad[1], "timeouts", bad[2], flush=True)
        if bad[0] == 0 and bad[1] == 0 and bad[2] == 0:
            print("FULL_SIZE_OK", flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
