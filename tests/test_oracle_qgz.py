"""Pins for the oracle's qgZ path: blockwise INT4 quantization and the
quantized all-to-all reduce-scatter.  CPU only."""
import numpy as np
import pytest

from oracle import hpz_oracle as O
from synth import inputs as S


def test_spec_constant_block():
    # ([2.0, 2.0, 2.0, 2.0], bits=8, block=4) -> scale=0, codes=[0,0,0,0], mins=[2.0]
    c, m, s = O.quantize_blockwise(np.full(4, 2.0, np.float32), bits=8, block=4)
    assert list(c) == [0, 0, 0, 0] and list(m) == [2.0] and list(s) == [0.0]
    # dequantize -> [2.0, 2.0] exactly
    assert list(O.dequantize_blockwise(c, m, s, block=4)) == [2.0] * 4


def test_spec_endpoints():
    # ([0.0, 1.0], bits=8, block=2) -> min=0, scale=1/255, codes=[0, 255]; round trip exact
    c, m, s = O.quantize_blockwise(np.array([0.0, 1.0], np.float32), bits=8, block=2)
    assert list(c) == [0, 255] and m[0] == 0.0 and s[0] == np.float32(1.0) / np.float32(255.0)
    v = O.dequantize_blockwise(c, m, s, block=2)
    assert v[0] == 0.0 and abs(v[1] - 1.0) <= 2 ** -23


@pytest.mark.parametrize("bits,block", [(4, 64), (8, 256)])
def test_error_bound_bruteforce(bits, block):
    """|v - v̂| <= scale/2 per element, with one fp32 rounding of slack."""
    rng = np.random.default_rng(bits)
    for scale in (1e-6, 1e-3, 1.0, 1e3):
        v = (rng.standard_normal(block * 200) * scale).astype(np.float32)
        c, m, s = O.quantize_blockwise(v, bits, block)
        assert c.max() <= (1 << bits) - 1
        vh = O.dequantize_blockwise(c, m, s, block)
        err = np.abs(v.astype(np.float64) - vh).reshape(-1, block)
        bound = s.astype(np.float64)[:, None] / 2 + 4 * np.abs(v).reshape(-1, block).max(axis=1, keepdims=True) * 2 ** -23
        assert np.all(err <= bound)


def test_monotone_codes():
    rng = np.random.default_rng(3)
    v = rng.standard_normal(64 * 50).astype(np.float32)
    c, m, s = O.quantize_blockwise(v)
    for b in range(50):
        order = np.argsort(v[b * 64:(b + 1) * 64], kind="stable")
        assert np.all(np.diff(c[b * 64:(b + 1) * 64][order].astype(int)) >= 0)


def test_nan_surfaces():
    v = np.zeros(128, np.float32)
    v[70] = np.nan
    c, m, s = O.quantize_blockwise(v)
    vh = O.dequantize_blockwise(c, m, s)
    assert np.all(np.isfinite(vh[:64])) and np.all(np.isnan(vh[64:]))


def test_qgz_rs_close_to_fp32_rs():
    P = 8
    lay = O.LayerLayout(50_000, P, 4, 256)
    G = [S.layer_grads(2, 1, j, lay.numel, lay.numel_pad) for j in range(P)]
    for r in range(P):
        q = O.qgz_reduce_scatter(G, lay, r).astype(np.float64)
        f = O.reduce_scatter(G, lay, r).astype(np.float64)
        s = lay.shard
        bound = np.zeros(s)
        for g in G:
            _, _, sc = O.quantize_blockwise(g)
            bound += np.repeat(sc[r * s // 64:(r + 1) * s // 64].astype(np.float64), 64) / 2
        assert np.all(np.abs(q - f) <= bound / P + 1e-9)


def test_qgz_rs_exact_on_constant_blocks():
    """Blocks constant per rank: quantization is exact, so qgZ == fp32 RS bitwise."""
    P = 4
    lay = O.LayerLayout(4096, P, 2, 256)
    G = [np.repeat((np.arange(lay.numel_pad // 64) % 7 - 3 + j).astype(np.float32) * 0.25, 64) for j in range(P)]
    for r in range(P):
        assert np.array_equal(O.qgz_reduce_scatter(G, lay, r), O.reduce_scatter(G, lay, r))


def test_qgz_payload_bytes():
    """int4 codes + fp32 (min, scale) per 64 elements = 0.625 B/elem vs 4 B/elem fp32."""
    assert O.QGZ_BITS / 8 + 8 / O.QGZ_BLOCK == 0.625


# ---------------------------------------------------------------- qwZ (f2)
def test_qwz_constant_blocks_exact():
    prim = O.bf16_rne(np.repeat(np.arange(8, dtype=np.float32) * 0.125 - 0.5, 256))
    assert np.array_equal(O.qwz_gathered_shard(prim, "bf16"), prim)


def test_qwz_error_bound():
    """Gathered weights within scale/2 + one bf16 rounding of the primary."""
    prim = O.bf16_rne(S.layer_params(0, 256 * 400))
    got = O.bf16_to_f32(O.qwz_gathered_shard(prim, "bf16")).astype(np.float64)
    ref = O.bf16_to_f32(prim).astype(np.float64)
    _, _, sc = O.quantize_blockwise(O.bf16_to_f32(prim), 8, 256)
    bound = np.repeat(sc.astype(np.float64), 256) / 2 + np.abs(ref) * 2 ** -8 + 1e-30
    assert np.all(np.abs(got - ref) <= bound)


def test_qwz_step_bwd_equals_fwd_and_trains():
    """hpZ + qwZ: the backward gather equals the (dequantized) forward gather, 0 mismatches."""
    o = O.HpzOracle([3000, 1234], 4, 2, align=256, qwz=True)
    for rec in o.run(3):
        assert sum(rec.mismatches) == 0
    # the forward-gathered weights differ from the exact primaries (lossy) but stay close
    prim = O.bf16_to_f32(o.full_primary(0)).astype(np.float64)
    assert np.max(np.abs(prim)) > 0
