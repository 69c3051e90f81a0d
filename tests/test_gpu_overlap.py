"""f3: the prefetch scheduler with real compute (paper_2407_01614_b200.overlap).

Single rank (P=1): the comm and compute streams of one rank overlap; libhpz's flags are
satisfied by the same rank's earlier kernels, so no kernel waits on a kernel it could
starve.  Checks: no-hpZ (off) and the fixed ordering train bit-identically (Fig. 2's
"no impact on model optimization"); the loss decreases; the stock ordering
with a delayed, poisoned secondary copy drives the loss to NaN (Table 1 'x')."""
import math

import pytest
import torch

from .gpu_util import gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a GPU")]


def _train(order, steps=6, depth=1, h=512, L=4, T=256):
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.overlap import PrefetchTrainer
    from paper_2407_01614_b200.world import EmulatedWorld, buffer_view
    from synth import inputs as S
    # stock needs a separate secondary to race on (at P' == P it is aliased to the primary)
    w = EmulatedWorld([h * h] * L, 1, 1, grad_dtype="bf16", timeout_s=10.0, alias_secondary=order != "stock")
    try:
        rc = w.ranks[0]
        H.hpz_set_order(rc.ctx, order, stock_delay_us=5000 if order == "stock" else 0,
                        stock_poison=order == "stock")
        H.hpz_set_option(rc.ctx, "max_ctas", 16)
        H.hpz_set_verify(rc.ctx, "fingerprint")
        s = torch.cuda.current_stream()
        for i in range(L):
            H.hpz_synth_master(rc.ctx, i, S.stream_key(S.SEED_PARAMS, i, 0, 0), 2.0 ** -5, s)
        g = torch.Generator(device="cuda").manual_seed(7)
        x = (torch.randn(T, h, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
        y = (torch.randn(T, h, device="cuda", generator=g) * 0.05).to(torch.bfloat16)
        tr = PrefetchTrainer(rc, h, L, T, depth=depth)
        losses = [float(tr.step(x, y)) for _ in range(steps)]
        torch.cuda.synchronize()
        master = [buffer_view(rc, i, "master", "f32").clone() for i in range(L)]
        c = H.hpz_counters(rc.ctx)
        return losses, master, c
    finally:
        w.close()


def test_fixed_equals_off_and_trains():
    lf, mf, cf = _train("fixed")
    lo, mo, _ = _train("off")
    assert lf == lo
    assert all(torch.equal(a.view(torch.int32), b.view(torch.int32)) for a, b in zip(mf, mo))
    assert lf[-1] < lf[0] and all(math.isfinite(v) for v in lf)
    assert cf["timeouts"] == 0 and cf["fp_mismatches"] == 0


def test_prefetch_depth_does_not_change_results():
    l1, m1, _ = _train("fixed", depth=1)
    l0, m0, _ = _train("fixed", depth=0)
    l2, m2, _ = _train("fixed", depth=2)
    assert l1 == l0 == l2


def test_stock_ordering_diverges():
    """Which stale secondary the backward reads is a hardware race: the poisoned one (NaN
    loss) or the previous step's (finite but wrong, caught by the fingerprints)."""
    ls, _, c = _train("stock", steps=4)
    assert any(not math.isfinite(v) for v in ls) or c["fp_mismatches"] > 0, (ls, c)


def _train_tf(order, steps=5, h=256, L=3, B=2, S=128, f=512, heads=4):
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.overlap import PrefetchTrainer, block_numel
    from paper_2407_01614_b200.world import EmulatedWorld
    from synth import inputs as S_
    w = EmulatedWorld([block_numel(h, f)] * L, 1, 1, grad_dtype="bf16", timeout_s=10.0,
                      alias_secondary=order != "stock")
    try:
        rc = w.ranks[0]
        H.hpz_set_order(rc.ctx, order, stock_delay_us=5000 if order == "stock" else 0,
                        stock_poison=order == "stock")
        H.hpz_set_option(rc.ctx, "max_ctas", 16)
        H.hpz_set_verify(rc.ctx, "fingerprint")
        s = torch.cuda.current_stream()
        for i in range(L):
            H.hpz_synth_master(rc.ctx, i, S_.stream_key(S_.SEED_PARAMS, i, 0, 0), 2.0 ** -5, s)
        g = torch.Generator(device="cuda").manual_seed(7)
        x = (torch.randn(B, S, h, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
        y = (x.float() * 0.05).to(torch.bfloat16)
        tr = PrefetchTrainer(rc, h, L, B * S, depth=1, model="transformer", ffn=f, n_heads=heads, lr=1e-4)
        losses = [float(tr.step(x, y)) for _ in range(steps)]
        torch.cuda.synchronize()
        return losses, H.hpz_counters(rc.ctx)
    finally:
        w.close()


def test_transformer_blocks_train_and_stock_diverges():
    """f3 with pre-norm transformer blocks (SDPA attention + GELU MLP, activation
    checkpointing): fixed and off agree (to attention-kernel rounding), the loss falls,
    the stock ordering with a poisoned delayed secondary goes NaN."""
    lf, cf = _train_tf("fixed")
    lo, _ = _train_tf("off")
    assert all(math.isfinite(v) for v in lf) and lf[-1] < lf[0], lf
    assert all(abs(a - b) <= 1e-3 * abs(b) for a, b in zip(lf, lo)), (lf, lo)
    assert cf["timeouts"] == 0 and cf["fp_mismatches"] == 0
    ls, cs = _train_tf("stock", steps=3)
    assert any(not math.isfinite(v) for v in ls) or cs["fp_mismatches"] > 0, (ls, cs)
