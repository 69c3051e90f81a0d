"""Pins for oracle a5 (reduce-scatter), a6 (Adam, bf16 refresh): CPU only."""
import json
import math
import os

import numpy as np
import pytest
import torch

from oracle import hpz_oracle as O
from synth import inputs as S

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- bf16 (R10)
def test_bf16_rne_golden():
    for src, dst in GOLD["bf16_rne"]["cases"]:
        x = np.array([int(src, 16)], dtype=np.uint32).view(np.float32)
        assert int(O.bf16_rne(x)[0]) == int(dst, 16), src


def test_bf16_rne_matches_torch_cast():
    """Special case that reduces to a library routine: torch's CPU fp32->bf16 cast is RNE."""
    rng = np.random.default_rng(0)
    x = np.concatenate([
        rng.standard_normal(200_000).astype(np.float32) * np.float32(1e-3),
        rng.integers(0, 2**32, 200_000, dtype=np.uint64).astype(np.uint32).view(np.float32),
    ])
    x = x[np.isfinite(x)]
    ours = O.bf16_rne(x)
    theirs = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, theirs)
    # NaN stays NaN (class, not payload)
    nan = np.array([np.nan, -np.nan], dtype=np.float32)
    assert np.all(O.is_nan_bits(O.bf16_rne(nan), "bf16"))


# ---------------------------------------------------------------- reduce-scatter
@pytest.mark.parametrize("ex", GOLD["reduce_scatter"])
def test_rs_spec_examples(ex):
    P = ex["P"]
    n = len(ex["grads"][0])
    lay = O.LayerLayout(n, P, 1 if P == 1 else P, 1)
    G = [np.array(g, dtype=np.float32) for g in ex["grads"]]
    for r in range(P):
        assert O.reduce_scatter(G, lay, r).tolist() == ex["shards"][r]


@pytest.mark.parametrize("P", [1, 2, 3, 4, 6, 8, 16])
def test_rs_dyadic_closed_form(P):
    """Dyadic-grid grads: every partial sum is exact in fp32, so the fixed-order result
    equals the exact rational mean (computed with Python integers)."""
    n = 4096
    lay = O.LayerLayout(n, P, 1, 1)
    G = [S.layer_grads(7, 3, r, n, kind="dyadic") for r in range(P)]
    ints = [np.round(g.astype(np.float64) * 2**20).astype(np.int64) for g in G]
    for r in range(P):
        got = O.reduce_scatter(G, lay, r)
        s = lay.shard
        exact = sum(int_g[r * s:(r + 1) * s] for int_g in ints)
        want = exact.astype(np.float64) / (2**20 * P)
        if P & (P - 1) == 0:
            assert np.array_equal(got.astype(np.float64), want)
        else:   # 1/P is inexact for non-powers of two: one rounding
            assert np.allclose(got, want, rtol=2**-23, atol=0)


def test_rs_error_bound_vs_float64():
    """|fl(sum) - sum| <= gamma_{ceil(log2 P)} * sum|G_j| for the pairwise tree (Higham §4.2)."""
    P = 8
    n = 50_000
    lay = O.LayerLayout(n, P, 4, 1)
    G = [S.layer_grads(0, 0, r, n) for r in range(P)]
    u = 2.0**-24
    depth = math.ceil(math.log2(P))
    gamma = depth * u / (1 - depth * u)
    for r in range(P):
        got = O.reduce_scatter(G, lay, r).astype(np.float64) * P
        s = lay.shard
        exact = sum(g[r * s:(r + 1) * s].astype(np.float64) for g in G)
        absum = sum(np.abs(g[r * s:(r + 1) * s].astype(np.float64)) for g in G)
        assert np.all(np.abs(got - exact) <= gamma * absum + 1e-45)


def test_rs_order_is_pairwise_tree():
    """Adversarial operands that distinguish the pairwise tree from a left fold:
    with G = [1, 2^-24, 2^-24, 2^-24]*... the tree keeps (2^-24+2^-24) = 2^-23 exact."""
    one, tiny = np.float32(1.0), np.float32(2.0**-24)
    G = [np.array([one]), np.array([tiny]), np.array([tiny]), np.array([tiny])]
    lay = O.LayerLayout(1, 4, 1, 1)
    # tree: (1 + 2^-24) + (2^-24 + 2^-24) = 1 + 2^-23 (ties-to-even 1+2^-24 -> 1, then 1 + 2^-23)
    got = O.reduce_scatter(G, lay, 0)[0] * 4
    assert got == np.float32(1.0 + 2.0**-23)
    # a left fold would give ((1 + 2^-24) + 2^-24) + 2^-24 = 1
    left = ((one + tiny) + tiny) + tiny
    assert left == np.float32(1.0)


def test_rs_dp_consistency():
    """Identical grads on all P ranks -> mean == the single-rank grad, bitwise."""
    for P in (1, 2, 4, 8, 16):
        n = 1000 * P
        lay = O.LayerLayout(n, P, 1, 1)
        g = S.layer_grads(1, 0, 0, n)
        G = [g.copy() for _ in range(P)]
        for r in range(P):
            assert np.array_equal(O.reduce_scatter(G, lay, r), g[r * lay.shard:(r + 1) * lay.shard])


# ---------------------------------------------------------------- Adam / SGD
def test_sgd_spec_example():
    ex = GOLD["sgd"]
    w = O.sgd_update(np.array(ex["w"], np.float32), np.array(ex["g"], np.float32), ex["lr"])
    assert np.allclose(w, ex["expect"], rtol=1e-7)


def test_adam_t1_closed_form():
    """At t=1: m̂=g, v̂=g², so Δw = -lr*g/(|g|+eps) (Kingma & Ba, bias-corrected)."""
    h = O.AdamHyper(lr=1e-3)
    g = S.layer_grads(0, 0, 0, 100_000)
    g = g[g != 0]
    w0 = np.zeros_like(g)
    w, m, v = O.adam_update(w0, np.zeros_like(g), np.zeros_like(g), g, O.adam_scalars(h, 1))
    g64 = g.astype(np.float64)
    want = -1e-3 * g64 / (np.abs(g64) + 1e-8)
    assert np.allclose(w.astype(np.float64), want, rtol=4e-6, atol=0)
    # "update magnitude ≈ lr regardless of g's scale"
    big = np.abs(g) > 1e-6          # |g| >> eps
    assert np.all(np.abs(np.abs(w[big]) - 1e-3) < 1e-3 * 0.02)


def test_adam_lr0_noop():
    h = O.AdamHyper(lr=0.0)
    w0 = S.layer_params(0, 4096)
    g = S.layer_grads(0, 0, 0, 4096)
    w, m, v = O.adam_update(w0, np.zeros_like(w0), np.zeros_like(w0), g, O.adam_scalars(h, 1))
    assert np.array_equal(w, w0)


@pytest.mark.parametrize("wd", [0.0, 0.01])
def test_adam_vs_torch_float64(wd):
    """vs torch.optim.Adam/AdamW in float64 over 5 steps: within 1e-6 relative."""
    n = 20_000
    h = O.AdamHyper(lr=1e-3, weight_decay=wd)
    w0 = S.layer_params(3, n)
    w, m, v = w0.copy(), np.zeros(n, np.float32), np.zeros(n, np.float32)
    p = torch.nn.Parameter(torch.from_numpy(w0.astype(np.float64)))
    opt = (torch.optim.AdamW([p], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, weight_decay=wd, foreach=False)
           if wd else torch.optim.Adam([p], lr=1e-3, betas=(0.9, 0.999), eps=1e-8, foreach=False))
    for t in range(5):
        g = S.layer_grads(3, t, 0, n)
        w, m, v = O.adam_update(w, m, v, g, O.adam_scalars(h, t + 1))
        p.grad = torch.from_numpy(g.astype(np.float64))
        opt.step()
    ref = p.detach().numpy()
    # fp32 storage vs float64: elementwise within 1e-6 relative to (|w| + lr), the
    # scale of one update; norm-wise within 1e-6 relative
    err = np.abs(w.astype(np.float64) - ref)
    assert np.all(err <= 1e-6 * (np.abs(ref) + 1e-3))
    assert np.linalg.norm(err) <= 1e-6 * np.linalg.norm(ref)


def test_adam_padding_stays_zero():
    h = O.AdamHyper()
    z = np.zeros(64, np.float32)
    w, m, v = O.adam_update(z, z, z, z, O.adam_scalars(h, 1))
    assert np.all(w == 0) and np.all(m == 0) and np.all(v == 0)


def test_adam_partitioned_equals_unpartitioned():
    """Adam over P shards == Adam over the concatenated vector, bitwise."""
    n, P = 8192, 8
    h = O.AdamHyper()
    lay = O.LayerLayout(n, P, 4, 1)
    w0 = S.layer_params(0, n)
    g = S.layer_grads(0, 0, 0, n)
    z = np.zeros(n, np.float32)
    wf, mf, vf = O.adam_update(w0, z, z, g, O.adam_scalars(h, 1))
    s = lay.shard
    parts = [O.adam_update(w0[r*s:(r+1)*s], z[:s], z[:s], g[r*s:(r+1)*s], O.adam_scalars(h, 1)) for r in range(P)]
    assert np.array_equal(np.concatenate([p[0] for p in parts]), wf)
    assert np.array_equal(np.concatenate([p[1] for p in parts]), mf)
    assert np.array_equal(np.concatenate([p[2] for p in parts]), vf)


def test_adam_scalars_validation():
    with pytest.raises(ValueError):
        O.adam_scalars(O.AdamHyper(), 0)


def test_bf16_grads_widen_exactly_and_rs_matches_float64_bound():
    """f4: bf16 gradient values widen to fp32 exactly (torch's cast agrees), and the
    fp32 fixed-order RS of the widened values obeys the pairwise error bound."""
    P = 8
    lay = O.LayerLayout(20_000, P, 4, 256)
    G = [S.layer_grads(0, 0, j, lay.numel, lay.numel_pad) for j in range(P)]
    Gb = [O.bf16_to_f32(O.bf16_rne(g)) for g in G]
    for g, gb in zip(G, Gb):
        tb = torch.from_numpy(g).to(torch.bfloat16).to(torch.float32).numpy()
        assert np.array_equal(tb.view(np.uint32), gb.view(np.uint32))
    u = 2.0 ** -24
    for r in range(P):
        got = O.reduce_scatter(Gb, lay, r).astype(np.float64) * P
        s = lay.shard
        exact = sum(g[r * s:(r + 1) * s].astype(np.float64) for g in Gb)
        absum = sum(np.abs(g[r * s:(r + 1) * s].astype(np.float64)) for g in Gb)
        assert np.all(np.abs(got - exact) <= 3 * u / (1 - 3 * u) * absum + 1e-45)
