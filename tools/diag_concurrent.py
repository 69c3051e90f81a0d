"""Diagnostic: emulated ranks on concurrent streams — where does parity break?"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from oracle import hpz_oracle as O
from tests.gpu_util import ParityRun, bits_np, bits_equal
from paper_2407_01614_b200 import hpz as H
from paper_2407_01614_b200.world import buffer_view

NUMELS = [300_007, 65_536, 4_099, 77]


def run_case(P, Pp, verify="fingerprint", ready_early=False, max_ctas=None, steps=3, sync_each_layer=False):
    run = ParityRun(NUMELS, P, Pp, fused=True, verify=verify)
    streams = [torch.cuda.Stream() for _ in range(P)]
    for rc in run.w.ranks:
        H.hpz_set_option(rc.ctx, "max_ctas", max_ctas or 144 // P)
    L = len(NUMELS)
    report = []
    for t in range(steps):
        grads = {(r, i): torch.from_numpy(np.ascontiguousarray(run.grads(i, t, r)[:run.o.layouts[i].numel])).cuda()
                 for r in range(P) for i in range(L)}
        torch.cuda.synchronize()
        for rc in run.w.ranks:
            s = streams[rc.rank]
            for i in range(L):
                H.hpz_fwd_gather(rc.ctx, i, run.fwd[rc.rank][i].data_ptr(), s)
            for i in reversed(range(L)):
                H.hpz_bwd_gather(rc.ctx, i, run.bwd[rc.rank][i].data_ptr(), s)
                H.hpz_grad_upload(rc.ctx, i, grads[(rc.rank, i)].data_ptr(), run.o.layouts[i].numel, s)
                if ready_early:
                    H.hpz_grads_ready(rc.ctx, i, s)
                H.hpz_reduce_scatter_adam(rc.ctx, i, run.adam, s)
        torch.cuda.synchronize()
        rec = run.o.step()
        run.t = t + 1
        for i, lay in enumerate(run.o.layouts):
            W = O.param_bits(rec.W[i], "bf16")
            G = [run.grads(i, t, j) for j in range(P)]
            Gp = [run.grads(i, t - 1, j) for j in range(P)] if t else None
            for r, rc in enumerate(run.w.ranks):
                f = bits_np(run.fwd[r][i], "bf16"); b = bits_np(run.bwd[r][i], "bf16")
                g = buffer_view(rc, i, "grad_shard", "f32").cpu().numpy()
                ref = O.reduce_scatter(G, lay, r)
                bad_rs = int(np.count_nonzero(g.view(np.uint32) != ref.view(np.uint32)))
                info = ""
                if bad_rs:
                    s_ = lay.shard
                    # which source ranks look stale: recompute with one rank's previous-step grads
                    for j in range(P):
                        if Gp is None: break
                        G2 = list(G); G2[j] = Gp[j]
                        alt = O.reduce_scatter(G2, lay, r)
                        m = int(np.count_nonzero(g.view(np.uint32) == alt.view(np.uint32)))
                        info += f" src{j}_prev_match={m}"
                    zero = [np.count_nonzero(g.view(np.uint32) == O.reduce_scatter([G[k] if k != j else np.zeros_like(G[k]) for k in range(P)], lay, r).view(np.uint32)) for j in range(P)]
                    info += f" src_zero_match={zero}"
                    idx = np.nonzero(g.view(np.uint32) != ref.view(np.uint32))[0]
                    info += f" first_bad={idx[:3].tolist()} last_bad={idx[-3:].tolist()} shard={s_}"
                nf = int(np.count_nonzero(f != W)); nb = int(np.count_nonzero(b != W))
                if nf or nb or bad_rs:
                    report.append(f"t={t} layer={i} rank={r} fwd_bad={nf} bwd_bad={nb} rs_bad={bad_rs}{info}")
    c = run.counters()
    run.close()
    return report, c


if __name__ == "__main__":
    for kw in [dict(P=4, Pp=2), dict(P=4, Pp=2, ready_early=True), dict(P=4, Pp=2, verify="none"),
               dict(P=4, Pp=2, max_ctas=8), dict(P=2, Pp=1), dict(P=4, Pp=4), dict(P=4, Pp=1)]:
        try:
            rep, c = run_case(**kw)
        except Exception as e:          # noqa: BLE001
            print(kw, "ERROR", e, flush=True)
            torch.cuda.synchronize()
            continue
        print(kw, "timeouts", c["timeouts"], "fp", c["fp_mismatches"], c["fp_fwd_mismatches"], "problems:", len(rep), flush=True)
        for line in rep[:12]:
            print("   ", line, flush=True)
