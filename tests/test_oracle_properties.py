"""Property-based pins of the oracle (hypothesis): invariants that must hold for every
topology and size, each tied to the paper / SPEC, not to the oracle's own code."""
import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import hpz_oracle as O
from synth import inputs as S

TOPO = st.sampled_from([(1, 1), (2, 1), (2, 2), (3, 1), (3, 3), (4, 2), (6, 3), (6, 2), (8, 4), (8, 1), (16, 4)])


@settings(max_examples=40, deadline=None)
@given(topo=TOPO, n=st.integers(1, 5000), align=st.sampled_from([1, 8, 64, 256]))
def test_layout_eq1_and_nesting(topo, n, align):
    """Eq. (1): s' = N̂/P' >= ceil(N/P'); secondary slice l == primaries l*k..l*k+k-1."""
    P, Pp = topo
    lay = O.LayerLayout(n, P, Pp, align)
    assert lay.numel_pad >= n and lay.numel_pad % (P * align) == 0 and lay.numel_pad - n < P * align
    assert lay.sec_shard * Pp == lay.numel_pad and lay.sec_shard >= -(-n // Pp)
    full = O.pad_full(np.arange(1, n + 1, dtype=np.float32), lay)
    prims = [O.partition_primary(full, lay, r) for r in range(P)]
    k = P // Pp
    for r in range(P):
        l = O.local_of(r, Pp)
        assert np.array_equal(O.secondary_copy(full, lay, r), np.concatenate(prims[l * k:(l + 1) * k]))


@settings(max_examples=25, deadline=None)
@given(topo=TOPO, layers=st.lists(st.integers(1, 3000), min_size=1, max_size=3), steps=st.integers(1, 2))
def test_fixed_order_never_stale(topo, layers, steps):
    """The paper's fix: the backward gather equals W_t bitwise for every topology (north_star)."""
    P, Pp = topo
    o = O.HpzOracle(layers, P, Pp, align=8)
    for rec in o.run(steps):
        assert sum(rec.mismatches) == 0 and sum(rec.nan_reads) == 0


@settings(max_examples=40, deadline=None)
@given(P=st.integers(1, 16), n=st.integers(1, 2000), seed=st.integers(0, 2 ** 31))
def test_rs_permutation_and_dyadic_exactness(P, n, seed):
    """Dyadic gradients: the fixed-order mean equals the exact rational mean, hence is
    invariant under any permutation of the ranks' contributions (commutativity check)."""
    lay = O.LayerLayout(n, P, 1, 1)
    G = [S.layer_grads(seed % 1000, 0, j, lay.numel, lay.numel_pad, kind="dyadic") for j in range(P)]
    perm = np.random.default_rng(seed).permutation(P)
    for r in range(P):
        a = O.reduce_scatter(G, lay, r)
        b = O.reduce_scatter([G[j] for j in perm], lay, r)
        if P & (P - 1) == 0:       # 1/P exact: both equal the exact mean
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32))
        else:
            assert np.allclose(a, b, rtol=2 ** -22, atol=0)


@settings(max_examples=40, deadline=None)
@given(scale=st.floats(1e-6, 1e6), seed=st.integers(0, 2 ** 31), bits=st.sampled_from([4, 8]))
def test_quantizer_bound(scale, seed, bits):
    """|v - dequant(quant(v))| <= scale_b/2 (+ fp32 rounding) for every element."""
    block = 64 if bits == 4 else 256
    v = (np.random.default_rng(seed).standard_normal(block * 4) * scale).astype(np.float32)
    c, m, s = O.quantize_blockwise(v, bits, block)
    vh = O.dequantize_blockwise(c, m, s, block).astype(np.float64)
    err = np.abs(v.astype(np.float64) - vh).reshape(-1, block)
    slack = 4 * np.abs(v).reshape(-1, block).max(axis=1, keepdims=True) * 2.0 ** -23
    assert np.all(err <= s.astype(np.float64)[:, None] / 2 + slack)
