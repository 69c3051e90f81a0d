"""GPU parity beyond the small fixed cases (VERDICT r1 "next" #2):

* layers large enough that every TMA CTA wraps its shared-memory stage ring several times
  at P >= 2 (the refill / parity-flip path of gather_tma_kernel and rs_tma_kernel), checked
  at sampled elements against the oracle's element-wise trajectory;
* special values — NaN, +-Inf, subnormals, -0, values whose reduction overflows — through the
  gathers, the reduce-scatter, Adam, qgZ and qwZ, compared with the oracle bit for bit with
  NaN compared by class (reading R10; NaN must surface, never vanish);
* the f3 prefetch trainer's optimizer steps replayed through the oracle from the gradients
  its GEMMs wrote.
"""
import numpy as np
import pytest
import torch

from oracle import hpz_oracle as O
from synth import inputs as S

from .gpu_util import ParityRun, bits_equal, bits_np, gpu_ok
from .test_gpu_parity import _check_step

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a GPU")]

F32 = np.float32


# ---------------------------------------------------------------- ring-wrapping sizes
@pytest.mark.parametrize("P,Pp,fused,engine", [(2, 1, True, "tma"), (4, 2, True, "tma"), (8, 4, True, "tma"),
                                               (4, 2, False, "tma"), (8, 4, True, "ldg"), (4, 4, True, "tma")])
def test_ring_wrapping_layer_sampled_parity(P, Pp, fused, engine):
    """One 21M-element layer: 1,282 RS chunks of 2,048 shard elements over <= 148 CTAs at
    P = 8 (~9 per CTA through a 2-6-stage ring), 41-164 gather chunks of 32 KiB per CTA.
    Three steps; forward and backward gathers of every rank, the reduced gradient shard and
    master / m / v / primary at ~4,000 sampled elements (incl. shard and chunk boundaries)
    against oracle.sampled_trajectory and the oracle's fixed-order sum."""
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import EmulatedWorld, buffer_view
    n, steps = 21_000_003, 3
    w = EmulatedWorld([n], P, Pp, timeout_s=30.0)
    try:
        s = torch.cuda.current_stream()
        info = w.ranks[0].infos[0]
        for rc in w.ranks:
            H.hpz_set_verify(rc.ctx, "fingerprint")
            H.hpz_set_option(rc.ctx, "copy_engine", H.COPY[engine])
            H.hpz_synth_master(rc.ctx, 0, S.stream_key(S.SEED_PARAMS, 0, 0, 0), S.PARAM_SCALE, s)
        fwd = [torch.empty(info.numel_pad, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        bwd = [torch.empty(info.numel_pad, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        rng = np.random.default_rng(5)
        edges = [0, n - 1, info.numel_pad - 1]
        for r in range(1, P):
            edges += [r * info.shard - 1, r * info.shard]
        for c in range(1, 40):
            edges += [c * 2048 - 1, c * 2048, c * 16384 - 1, c * 16384]
        idx = np.unique(np.concatenate([rng.integers(0, info.numel_pad, 4000), np.array(edges)]))
        idx_t = torch.from_numpy(idx).cuda()
        adam = H.make_adam()
        hyper = O.AdamHyper()
        for t in range(steps):
            _, _, _, p_t = O.sampled_trajectory(0, n, P, idx, t, hyper)
            for rc in w.ranks:
                H.hpz_fwd_gather(rc.ctx, 0, fwd[rc.rank].data_ptr(), s)
            for rc in w.ranks:
                H.hpz_bwd_gather(rc.ctx, 0, bwd[rc.rank].data_ptr(), s)
            for rc in w.ranks:
                H.hpz_synth_grads(rc.ctx, 0, S.stream_key(S.SEED_GRADS, 0, t, rc.rank), S.GRAD_SCALE, 0, s)
            for rc in w.ranks:
                H.hpz_grads_ready(rc.ctx, 0, s)
            for rc in w.ranks:
                (H.hpz_reduce_scatter_adam(rc.ctx, 0, adam, s) if fused else H.hpz_reduce_scatter(rc.ctx, 0, s))
            if not fused:
                for rc in w.ranks:
                    H.hpz_step(rc.ctx, -1, adam, s)
            torch.cuda.synchronize()
            for r in range(P):
                assert np.array_equal(bits_np(fwd[r][idx_t], "bf16"), p_t), (t, r, "fwd")
                assert np.array_equal(bits_np(bwd[r][idx_t], "bf16"), p_t), (t, r, "bwd")
        wt, m, v, p = O.sampled_trajectory(0, n, P, idx, steps, hyper)
        g_last = (O.pairwise_rank_sum([S.values_at(S.SEED_GRADS, 0, steps - 1, r, idx, S.GRAD_SCALE, n)
                                       for r in range(P)]) * F32(1.0 / P)).astype(F32)
        for rc in w.ranks:
            lo, hi = rc.rank * info.shard, (rc.rank + 1) * info.shard
            sel = (idx >= lo) & (idx < hi)
            loc = torch.from_numpy(idx[sel] - lo).cuda()
            for kind, ref in (("master", wt), ("m", m), ("v", v), ("grad_shard", g_last)):
                got = buffer_view(rc, 0, kind, "f32")[loc].cpu().numpy()
                assert np.array_equal(got.view(np.uint32), ref[sel].view(np.uint32)), (rc.rank, kind)
            got = bits_np(buffer_view(rc, 0, "primary", "bf16")[loc], "bf16")
            assert np.array_equal(got, p[sel]), (rc.rank, "primary")
        c = [H.hpz_counters(rc.ctx) for rc in w.ranks]
        assert sum(x["timeouts"] + x["fp_mismatches"] + x["fp_fwd_mismatches"] for x in c) == 0, c
        assert sum(x["fp_fwd_checked"] for x in c) == steps * P
    finally:
        w.close()


# ---------------------------------------------------------------- special values
NUMELS = [70_001, 4_099]


def _special_params(i, n):
    rng = np.random.default_rng(100 + i)
    w = (rng.standard_normal(n) * 0.02).astype(F32)
    k = rng.permutation(n)
    w[k[0:50]] = F32(0.0)
    w[k[50:100]] = F32(-0.0)
    w[k[100:200]] = (rng.standard_normal(100) * 1e-40).astype(F32)       # fp32 subnormals
    w[k[200:250]] = (rng.standard_normal(50) * 1e-39).astype(F32)        # below bf16's normal range
    w[k[250:300]] = (rng.standard_normal(50) * 3e38).astype(F32)         # near fp32 max (bf16 overflow)
    w[k[300:303]] = [np.inf, -np.inf, np.nan]
    return w


def _special_grads(t, r, i):
    n = NUMELS[i]
    rng = np.random.default_rng(1000 * t + 10 * r + i)
    g = (rng.standard_normal(n) * 1e-3).astype(F32)
    k = np.random.default_rng(7 + i).permutation(n)       # same positions on every rank
    g[k[0:40]] = np.nan if r == 0 else g[k[0:40]]          # NaN from one rank only
    g[k[40:80]] = np.inf if r % 2 == 0 else -np.inf        # +inf + -inf = NaN in the sum
    g[k[80:120]] = np.inf                                   # +inf everywhere
    g[k[120:220]] = (np.random.default_rng(t + r).standard_normal(100) * 1e-42).astype(F32)   # subnormal grads
    g[k[220:260]] = F32(-0.0)
    g[k[260:300]] = F32(3e38)                               # the sum overflows to inf
    g[k[300 + 64 * t:364 + 64 * t]] = np.nan                # a whole qgZ block NaN, moving per step
    return g


@pytest.mark.parametrize("P,Pp,kw", [(1, 1, {}), (4, 2, {}), (8, 4, {"fused": False}), (4, 2, {"qgz": True}),
                                     (4, 2, {"qwz": True}), (4, 2, {"grad_dtype": "bf16"}),
                                     (2, 1, {"dtype": "f32"}), (4, 2, {"copy_engine": "ldg", "verify": "exact"})])
def test_special_values_parity(P, Pp, kw):
    """NaN / Inf / subnormal / -0 / overflowing values through every stage, bit-exact vs the
    oracle with NaN compared by class: NaN in a gradient surfaces in the reduced shard and in
    the updated master / primary of those elements, inf + -inf -> NaN,
    overflow -> inf, subnormals survive the fp32 arithmetic and the bf16 rounding."""
    kw = dict(kw)
    fused = kw.pop("fused", True)
    run = ParityRun(NUMELS, P, Pp, fused=fused, init_params=[_special_params(i, n) for i, n in enumerate(NUMELS)],
                    grad_override=_special_grads, **{"verify": "fingerprint", **kw})
    try:
        for _ in range(3):
            _check_step(run, run.step())
        c = run.counters()
        assert c["timeouts"] == 0, c
    finally:
        run.close()


def test_special_values_reach_the_outputs():
    """The special-value case is not vacuous: NaN and inf reach the reduced shard and the
    updated master in both the oracle and the GPU."""
    run = ParityRun(NUMELS, 4, 2, fused=True, init_params=[_special_params(i, n) for i, n in enumerate(NUMELS)],
                    grad_override=_special_grads, verify="fingerprint")
    try:
        _check_step(run, run.step())
        from paper_2407_01614_b200.world import buffer_view
        g = np.concatenate([buffer_view(rc, 0, "grad_shard", "f32").cpu().numpy() for rc in run.w.ranks])
        mst = np.concatenate([buffer_view(rc, 0, "master", "f32").cpu().numpy() for rc in run.w.ranks])
        assert np.isnan(g).sum() >= 80 and np.isinf(g).sum() >= 40
        assert np.isnan(mst).sum() >= 80
        sub = (np.abs(g) > 0) & (np.abs(g) < np.finfo(F32).tiny)
        assert sub.sum() > 0
    finally:
        run.close()


# ---------------------------------------------------------------- f3 vs the oracle
@pytest.mark.parametrize("model", ["mlp", "transformer"])
def test_prefetch_trainer_steps_replayed_by_oracle(model):
    """Alg. 1's PrefetchAllGather around real GEMMs (paper_2407_01614_b200.overlap): after
    every training step, the gradient slots the backward GEMMs wrote are fed to the oracle,
    whose reduce-scatter + Adam must reproduce the trainer's master / m / v / primary bit for
    bit — the prefetching scheduler moved the right parameters of the right step through the
    library."""
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.overlap import PrefetchTrainer, block_numel
    from paper_2407_01614_b200.world import EmulatedWorld, buffer_view
    h, L = (512, 4) if model == "mlp" else (256, 3)
    f, heads, B, Sq = 512, 4, 2, 128
    n = h * h if model == "mlp" else block_numel(h, f)
    numels = [n] * L
    w = EmulatedWorld(numels, 1, 1, grad_dtype="bf16", timeout_s=10.0)
    captured = {}
    o = O.HpzOracle(numels, 1, 1, grad_dtype="bf16", grad_override=lambda t, r, i: captured[(t, i)])
    try:
        rc = w.ranks[0]
        H.hpz_set_option(rc.ctx, "max_ctas", 16)
        H.hpz_set_verify(rc.ctx, "fingerprint")
        s = torch.cuda.current_stream()
        for i in range(L):
            H.hpz_synth_master(rc.ctx, i, S.stream_key(S.SEED_PARAMS, i, 0, 0), S.PARAM_SCALE, s)
        g = torch.Generator(device="cuda").manual_seed(7)
        if model == "mlp":
            x = (torch.randn(256, h, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
            y = (torch.randn(256, h, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
            tr = PrefetchTrainer(rc, h, L, 256, depth=1)
        else:
            x = (torch.randn(B, Sq, h, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
            y = (x.float() * 0.05).to(torch.bfloat16)
            tr = PrefetchTrainer(rc, h, L, B * Sq, depth=1, model="transformer", ffn=f, n_heads=heads)
        for t in range(3):
            tr.step(x, y)
            torch.cuda.synchronize()
            for i in range(L):
                captured[(t, i)] = tr.gslots[i][:n].float().cpu().numpy()
            o.step()
            for i in range(L):
                st = o.state[i][0]
                for kind, ref in (("master", st.master), ("m", st.m), ("v", st.v)):
                    got = buffer_view(rc, i, kind, "f32").cpu().numpy()
                    assert bits_equal(got.view(np.uint32), ref.view(np.uint32), "f32"), (model, t, i, kind)
                got = bits_np(buffer_view(rc, i, "primary", "bf16"), "bf16")
                assert bits_equal(got, O.param_bits(st.prim, "bf16"), "bf16"), (model, t, i, "primary")
        c = H.hpz_counters(rc.ctx)
        assert c["timeouts"] == 0 and c["fp_mismatches"] == 0 and c["fp_fwd_mismatches"] == 0, c
    finally:
        w.close()
