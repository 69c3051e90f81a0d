"""Pins for the oracle's whole step (Alg. 1) and a7 (stale-param
mismatch), incl. the deliberately re-introduced stock ordering.  CPU only."""
import numpy as np
import pytest

from oracle import hpz_oracle as O

SMALL = [3000, 1234, 777]


def _params_equal(a: O.HpzOracle, b: O.HpzOracle):
    for i in range(len(a.layouts)):
        if not np.array_equal(a.full_master(i).view(np.uint32), b.full_master(i).view(np.uint32)):
            return False
    return True


@pytest.mark.parametrize("P,Pp", [(1, 1), (2, 1), (2, 2), (4, 2), (8, 4), (8, 2), (8, 1), (8, 8)])
def test_fixed_zero_mismatch_and_bwd_equals_fwd(P, Pp):
    """Fixed ordering: the backward gather equals W_t bitwise (north_star invariant)."""
    o = O.HpzOracle(SMALL, P, Pp, align=16, order="fixed")
    for rec in o.run(3):
        assert sum(rec.mismatches) == 0 and sum(rec.nan_reads) == 0


def test_secondary_equals_primary_slice_after_every_step():
    """R11: after fwd(t) the secondary equals the matching slice of the primaries as of W_t."""
    o = O.HpzOracle(SMALL, 8, 4, align=16)
    for _ in range(3):
        prims_before = [[o.state[i][r].prim.copy() for r in range(8)] for i in range(3)]
        o.step()
        for i, lay in enumerate(o.layouts):
            k = 8 // 4
            for r in range(8):
                l = O.local_of(r, 4)
                assert np.array_equal(o.state[i][r].sec, np.concatenate(prims_before[i][l * k:(l + 1) * k]))


def test_padding_stays_zero():
    o = O.HpzOracle(SMALL, 8, 4, align=256)
    o.run(3)
    for i, lay in enumerate(o.layouts):
        assert np.all(o.full_master(i)[lay.numel:] == 0)
        assert np.all(o.full_primary(i)[lay.numel:] == 0)


def test_scheme_equivalence_synthetic():
    """fixed == off == stock-under-program-order, bit-identical params."""
    runs = [O.HpzOracle(SMALL, 8, 4, align=16, order=o_, stock_schedule="program") for o_ in ("fixed", "off", "stock")]
    for r in runs:
        r.run(3)
    assert _params_equal(runs[0], runs[1]) and _params_equal(runs[0], runs[2])


def test_partitioned_equals_unpartitioned_adam_and_sgd():
    """Brute force against unpartitioned training on the whole vector (north_star)."""
    for opt in ("adam", "sgd"):
        o = O.HpzOracle(SMALL, 8, 4, align=16, optimizer=opt, param_dtype="f32")
        o.run(4)
        master, _, _, _ = O.unpartitioned_train(SMALL, 8, 4, O.AdamHyper(), param_dtype="f32", optimizer=opt)
        for i, lay in enumerate(o.layouts):
            assert np.array_equal(o.full_master(i)[:lay.numel], master[i]), (opt, i)


def test_stock_adversarial_stale_closed_form():
    """Stock + adversarial schedule: at t=0 every element is poison (NaN); at t>=1 the
    backward gather returns W_{t-1}, so mismatches == P * #{e: bits(W_t) != bits(W_{t-1})}."""
    P, Pp = 8, 4
    o = O.HpzOracle(SMALL, P, Pp, align=16, order="stock", stock_schedule="adversarial_stale")
    recs = o.run(3)
    for i, lay in enumerate(o.layouts):
        assert recs[0].mismatches[i] == P * lay.numel
        assert recs[0].nan_reads[i] == P * lay.numel
    for t in (1, 2):
        for i, lay in enumerate(o.layouts):
            cur = O.param_bits(recs[t].W[i], "bf16")[:lay.numel]
            prev = O.param_bits(recs[t - 1].W[i], "bf16")[:lay.numel]
            expect = P * int(np.count_nonzero(cur != prev))
            assert recs[t].mismatches[i] == expect
            assert expect > 0


def test_stock_realloc_reads_poison():
    """Paper-faithful realloc (torch.empty each step): every read is NaN."""
    o = O.HpzOracle(SMALL, 8, 2, align=16, order="stock", stock_schedule="realloc")
    for rec in o.run(2):
        for i, lay in enumerate(o.layouts):
            assert rec.nan_reads[i] == 8 * lay.numel == rec.mismatches[i]


def test_stock_half_written_mismatch_positive():
    o = O.HpzOracle(SMALL, 8, 4, align=16, order="stock", stock_schedule="half_written")
    recs = o.run(3)
    assert sum(recs[0].mismatches) > 0
    assert sum(sum(r.mismatches) for r in recs) > 0


def test_stock_does_not_change_synthetic_trajectory():
    """With parameter-independent synthetic grads the race only shows in the counters."""
    a = O.HpzOracle(SMALL, 8, 4, align=16, order="fixed")
    b = O.HpzOracle(SMALL, 8, 4, align=16, order="stock", stock_schedule="adversarial_stale")
    a.run(2)
    b.run(2)
    assert _params_equal(a, b)


# ---------------------------------------------------------------- toy MLP (config C1)
def test_toy_param_count():
    assert sum(O.toy_layer_numels((4, 8, 2))) == 58
    assert O.toy_layer_numels() == [525312, 524800]            # BASELINE C1: 1,050,112


def test_toy_grads_vs_finite_differences():
    """Reverse-mode grads within 1e-4 relative of central finite differences."""
    dims = (6, 5, 3)
    rng = np.random.default_rng(0)
    flat = [rng.standard_normal(n) * 0.5 for n in O.toy_layer_numels(dims)]
    x = rng.standard_normal((4, 6))
    y = rng.standard_normal((4, 3))
    loss, grads = O.toy_loss_and_grads(flat, flat, x, y, dims)
    h = 1e-6
    for li in range(2):
        for e in range(flat[li].size):
            fp = [f.copy() for f in flat]
            fm = [f.copy() for f in flat]
            fp[li][e] += h
            fm[li][e] -= h
            num = (O.toy_loss_and_grads(fp, fp, x, y, dims)[0] - O.toy_loss_and_grads(fm, fm, x, y, dims)[0]) / (2 * h)
            assert abs(num - grads[li][e]) <= 1e-4 * max(abs(num), 1e-3), (li, e)


def test_toy_zero_weights_zero_targets():
    dims = (4, 8, 2)
    flat = [np.zeros(n) for n in O.toy_layer_numels(dims)]
    x = np.ones((3, 4))
    loss, grads = O.toy_loss_and_grads(flat, flat, x, np.zeros((3, 2)), dims)
    assert loss == 0 and all(np.all(g == 0) for g in grads)


@pytest.fixture(scope="module")
def toy_runs():
    """Config C1: toy 2-layer MLP, 1,050,112 fp32 params, 8 ranks as 2x4, 5 Adam steps."""
    numels = O.toy_layer_numels()
    out = {}
    for name, kw in {"fixed": dict(order="fixed"), "off": dict(order="off"),
                     "stock_prog": dict(order="stock", stock_schedule="program"),
                     "stock_adv": dict(order="stock", stock_schedule="adversarial_stale")}.items():
        o = O.HpzOracle(numels, 8, 4, align=256, param_dtype="f32", grad_source="toy",
                        hyper=O.AdamHyper(lr=1e-3), **kw)
        recs = o.run(5)
        out[name] = (o, recs)
    return out


def test_toy_c1_fixed_converges_and_matches_off(toy_runs):
    o_fix, r_fix = toy_runs["fixed"]
    o_off, r_off = toy_runs["off"]
    o_sp, r_sp = toy_runs["stock_prog"]
    losses = [r.loss for r in r_fix]
    assert losses[-1] < losses[0]                       # training loss decreases
    assert [r.loss for r in r_off] == losses            # Fig. 2: no-hpZ == modified hpZ
    assert [r.loss for r in r_sp] == losses
    assert _params_equal(o_fix, o_off) and _params_equal(o_fix, o_sp)
    assert all(sum(r.mismatches) == 0 for r in r_fix)


def test_toy_c1_stock_goes_nan_and_stays(toy_runs):
    """Table 1 '×': stock hpZ under the adversarial schedule -> NaN loss, and NaN is
    monotone afterwards."""
    _, recs = toy_runs["stock_adv"]
    assert sum(recs[0].mismatches) > 0
    first_nan = next(i for i, r in enumerate(recs) if not np.isfinite(r.loss))
    assert all(not np.isfinite(r.loss) for r in recs[first_nan:])


def test_toy_c1_matches_unpartitioned(toy_runs):
    o_fix, r_fix = toy_runs["fixed"]
    master, _, _, losses = O.unpartitioned_train(O.toy_layer_numels(), 8, 5, O.AdamHyper(lr=1e-3),
                                                 param_dtype="f32", grad_source="toy",
                                                 init_full=[o_fix.history[0].W[i][:n].astype(np.float32)
                                                            for i, n in enumerate(O.toy_layer_numels())])
    assert losses == [r.loss for r in r_fix]
    for i, lay in enumerate(o_fix.layouts):
        assert np.array_equal(o_fix.full_master(i)[:lay.numel], master[i])


def test_toy_dp_consistency():
    """Identical batches on all ranks: the P-rank run equals the 1-rank run bitwise."""
    numels = O.toy_layer_numels((16, 32, 8))
    # toy_batch uses TOY_DIMS; use the default dims with identical batches, 2 steps
    numels = O.toy_layer_numels()
    a = O.HpzOracle(numels, 4, 2, align=256, param_dtype="f32", grad_source="toy", toy_identical_batches=True)
    b = O.HpzOracle(numels, 1, 1, align=256, param_dtype="f32", grad_source="toy", toy_identical_batches=True)
    a.run(2)
    b.run(2)
    for i, lay in enumerate(a.layouts):
        assert np.array_equal(a.full_master(i)[:lay.numel], b.full_master(i)[:lay.numel])


def test_sampled_trajectory_matches_full_sim():
    """The per-element sampled evaluation used at BASELINE sizes equals the full simulation."""
    o = O.HpzOracle([5000], 4, 2, align=16)
    o.run(3)
    idx = np.array([0, 1, 17, 2048, 4999, 5000 - 1])
    w, m, v, p = O.sampled_trajectory(0, 5000, 4, idx, 3, O.AdamHyper())
    assert np.array_equal(w, o.full_master(0)[idx])
    assert np.array_equal(p, o.full_primary(0)[idx])


def test_realistic_racing_layers_closed_form():
    """Alg. 1's enqueue order with prefetch depth d: the backward gathers
    enqueued before their layer's secondary copy are exactly the last ceil(d/2) layers —
    the forward->backward turnaround of Fig. 1 — and none without prefetch.
    Derivation: bwd L_j (1-based) is module 2N+1-j, prefetched while module 2N+1-j-d runs;
    its copy follows module j, so it races iff 2N+1-j-d <= j, i.e. j >= N - (d-1)/2."""
    import math
    for N in range(1, 8):
        for d in range(0, 15):
            k = min(N, math.ceil(d / 2))
            assert O.realistic_racing_layers(N, d) == set(range(N - k, N)), (N, d)
    # the program order itself: every gather is enqueued once, every copy after its forward
    seq = O.prefetch_enqueue_order(4, 1)
    assert sorted(x for x in seq if x[0] == "gather") == sorted(
        [("gather", "fwd", i) for i in range(4)] + [("gather", "bwd", i) for i in range(4)])
    assert seq.index(("gather", "fwd", 2)) < seq.index(("copy", 1)) < seq.index(("gather", "fwd", 3))
    assert seq.index(("gather", "bwd", 3)) < seq.index(("copy", 3))        # the turnaround race


@pytest.mark.parametrize("depth", [1, 3])
def test_stock_realistic_closed_form(depth):
    """Stock + realistic schedule: only the racing layers read stale data — poison at t=0
    (every element NaN), W_{t-1} afterwards (mismatches = P * #{e: W_t[e] != W_{t-1}[e]});
    every other layer reads its fresh copy (0 mismatches); fixed ordering reads nothing stale."""
    P, Pp = 4, 2
    numels = [3000, 2500, 4096, 77, 1234]
    racing = O.realistic_racing_layers(len(numels), depth)
    assert racing == ({4} if depth == 1 else {3, 4})
    o = O.HpzOracle(numels, P, Pp, align=16, order="stock", stock_schedule="realistic", prefetch_depth=depth)
    recs = o.run(3)
    for t, rec in enumerate(recs):
        for i, lay in enumerate(o.layouts):
            if i not in racing:
                assert rec.mismatches[i] == 0 and rec.nan_reads[i] == 0, (t, i)
            elif t == 0:
                assert rec.mismatches[i] == P * lay.numel == rec.nan_reads[i], (t, i)
            else:
                cur = O.param_bits(rec.W[i], "bf16")[:lay.numel]
                prev = O.param_bits(recs[t - 1].W[i], "bf16")[:lay.numel]
                assert rec.mismatches[i] == P * int(np.count_nonzero(cur != prev)) > 0, (t, i)
    f = O.HpzOracle(numels, P, Pp, align=16, order="fixed", stock_schedule="realistic", prefetch_depth=depth)
    assert all(sum(r.mismatches) == 0 for r in f.run(2))
