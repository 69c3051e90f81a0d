#!/usr/bin/env python
"""Step-by-step probe of the push reduce-scatter in single-GPU emulation (P=2): every call
is followed by a synchronize, then the landing counters / RL_FREE / slot flags are read
from the arenas (control-region layout of hpz_runtime.cpp's register)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2407_01614_b200 import hpz as H  # noqa: E402
from paper_2407_01614_b200.world import EmulatedWorld, device_view  # noqa: E402
from synth import inputs as S  # noqa: E402


def a256(x):
    return (x + 255) // 256 * 256


def main():
    P, numels = 2, [300_007]
    W = EmulatedWorld(numels, P, 1, timeout_s=3.0, rs_push=True)
    L, Sl, n_land, kRsl = len(numels), len(numels), 0, 2
    n_flags = 5 * L * P + 2 * Sl * P + 2 * n_land * P + kRsl * P
    off_ctr = a256(n_flags * 4)
    off_fp = a256(off_ctr + 7 * (L + Sl) * 4)
    off_stats = a256(off_fp + L * 32)
    off_rsc = a256(off_stats + 64)
    shard = W.ranks[0].infos[0].shard
    chunks = (shard + 2047) // 2048
    s = torch.cuda.current_stream()

    def u32(rank, off, n):
        return device_view(H.hpz_arena_ptr(W.ranks[rank].ctx, rank) + off, n, "f32").view(torch.int32).cpu().tolist()

    def show(tag):
        torch.cuda.synchronize()
        for r in range(P):
            fl = u32(r, 0, n_flags)
            rl = fl[5 * L * P + 2 * Sl * P:]
            rs_done = fl[5 * L * P + Sl * P: 5 * L * P + 2 * Sl * P]
            ctr = u32(r, off_rsc, 2 * chunks)
            print(f"[{tag}] rank {r}: err={H.hpz_last_error(W.ranks[r].ctx)!r} RL_FREE={rl} RS_DONE={rs_done} "
                  f"rsc0[:6]={ctr[:6]} rsc0 sum={sum(ctr[:chunks])} rsc1 sum={sum(ctr[chunks:])} (chunks {chunks})",
                  flush=True)
        c = H.hpz_counters(W.ranks[0].ctx)
        print(f"[{tag}] timeouts={c['timeouts']}", flush=True)

    w0 = torch.from_numpy(S.layer_params(0, numels[0])).cuda()
    outs = [torch.empty(W.ranks[0].infos[0].numel_pad, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
    for rc in W.ranks:
        H.hpz_load_master(rc.ctx, 0, w0.data_ptr(), s)
    adam = H.make_adam()
    for step in range(2):
        for rc in W.ranks:
            H.hpz_fwd_gather(rc.ctx, 0, outs[rc.rank].data_ptr(), s)
        show(f"t{step} fwd")
        for rc in W.ranks:
            H.hpz_bwd_gather(rc.ctx, 0, outs[rc.rank].data_ptr(), s)
        show(f"t{step} bwd")
        for rc in W.ranks:
            H.hpz_synth_grads(rc.ctx, 0, S.stream_key(S.SEED_GRADS, 0, step, rc.rank), S.GRAD_SCALE, 0, s)
        show(f"t{step} grads")
        for rc in W.ranks:
            H.hpz_grads_ready(rc.ctx, 0, s)
            show(f"t{step} push r{rc.rank}")
        for rc in W.ranks:
            H.hpz_reduce_scatter_adam(rc.ctx, 0, adam, s)
            show(f"t{step} reduce r{rc.rank}")
    W.close()


if __name__ == "__main__":
    main()
