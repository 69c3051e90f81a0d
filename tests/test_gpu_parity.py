"""GPU parity: the CUDA path through the C ABI vs the CPU oracle, element by element.

Ranks are emulated in one process on one GPU (paper_2407_01614_b200.world.EmulatedWorld),
so every (P, P') of BASELINE.json's sweep is covered on a single B200; the real
multi-process NVLink path is covered by tests/test_gpu_multiproc.py when >= 2 GPUs exist.
Bars (north_star): gathers, secondaries, shard indexing and the fp32 reduce-scatter
bit-exact; Adam within 1e-6 relative (the kernel matches the oracle's op sequence, so
the test asserts bit-exactness and reports the max relative error on failure).
"""
import numpy as np
import pytest
import torch

from oracle import hpz_oracle as O
from synth import inputs as S

from .gpu_util import ParityRun, bits_equal, bits_np, gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a GPU")]

# several 32 KiB gather tiles per shard plus ragged tails; one layer smaller than P*A
NUMELS = [300_007, 65_536, 4_099, 77]
TOPOS = [(1, 1), (2, 1), (2, 2), (4, 1), (4, 2), (4, 4), (8, 1), (8, 2), (8, 4), (8, 8)]


def _check_step(run: ParityRun, rec, check_all=True, check_secondary=True):
    P, dtype = run.P, run.dtype
    for i, lay in enumerate(run.o.layouts):
        W = O.param_bits(rec.W[i], dtype)
        for r, rc in enumerate(run.w.ranks):
            # a2: forward gather == W_t bitwise (incl. zero padding; NaN by class, R10)
            assert bits_equal(bits_np(run.fwd[r][i], dtype), W, dtype), f"fwd layer {i} rank {r}"
            # a4: backward gather == W_t bitwise
            assert bits_equal(bits_np(run.bwd[r][i], dtype), W, dtype), f"bwd layer {i} rank {r}"
        if not check_all:
            continue
        from paper_2407_01614_b200.world import buffer_view
        grads = [run.grads(i, run.t - 1, j) for j in range(P)]
        if run.grad_dtype == "bf16":
            grads = [O.bf16_to_f32(O.bf16_rne(g)) for g in grads]
        for r, rc in enumerate(run.w.ranks):
            st = run.o.state[i][r]
            # a2 secondary store == oracle's Eq. (1) slice; at P' == P the library aliases the
            # secondary to the primary, which after the step holds W_{t+1}
            aliased = run.Pp == P and not run.qwz
            if run.o.order == "fixed" and check_secondary:   # (paper maps to fixed)
                sec = bits_np(buffer_view(rc, i, "secondary", dtype), dtype)
                want = st.prim if aliased else st.sec
                assert bits_equal(sec, O.param_bits(want, dtype), dtype), f"secondary layer {i} rank {r}"
            # a5 reduce-scatter bit-exact in the fixed order
            if run.store_grad_shard:
                g_gpu = buffer_view(rc, i, "grad_shard", "f32").cpu().numpy()
                g_ref = (O.qgz_reduce_scatter if run.qgz else O.reduce_scatter)(grads, lay, r)
                assert bits_equal(g_gpu.view(np.uint32), g_ref.view(np.uint32), "f32"), f"RS layer {i} rank {r}"
            # a6 Adam + bf16 refresh
            for kind, ref in (("master", st.master), ("m", st.m), ("v", st.v)):
                got = buffer_view(rc, i, kind, "f32").cpu().numpy()
                if not bits_equal(got.view(np.uint32), ref.view(np.uint32), "f32"):
                    rel = np.nanmax(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-30))
                    pytest.fail(f"{kind} layer {i} rank {r}: max rel err {rel:.3g}")
            prim = bits_np(buffer_view(rc, i, "primary", dtype), dtype)
            assert bits_equal(prim, O.param_bits(st.prim, dtype), dtype), f"primary layer {i} rank {r}"


ENGINES = [("ldg", "exact"), ("tma", "fingerprint")]   # EXACT verification runs on the LDG kernel


@pytest.mark.parametrize("engine,verify", ENGINES)
@pytest.mark.parametrize("P,Pp", TOPOS)
def test_parity_fixed(P, Pp, engine, verify):
    run = ParityRun(NUMELS, P, Pp, copy_engine=engine, verify=verify)
    try:
        for _ in range(3):
            rec = run.step()
            _check_step(run, rec)
        c = run.counters()
        assert c["mismatches"] == 0 and c["nan_reads"] == 0 and c["timeouts"] == 0
        assert c["fp_mismatches"] == 0 and c["fp_checked"] == 3 * len(NUMELS) * P
    finally:
        run.close()


@pytest.mark.parametrize("engine,verify", ENGINES)
@pytest.mark.parametrize("P,Pp", TOPOS)
@pytest.mark.parametrize("store", [True, False])
def test_parity_fused_rs_adam(P, Pp, store, engine, verify):
    """hpz_reduce_scatter_adam == hpz_reduce_scatter + hpz_step, bit for bit."""
    if not store and P not in (1, 8):
        pytest.skip("store=False covered at P=1, 8")
    run = ParityRun(NUMELS, P, Pp, fused=True, store_grad_shard=store, copy_engine=engine, verify=verify)
    try:
        for _ in range(3):
            _check_step(run, run.step())
        c = run.counters()
        assert c["mismatches"] == 0 and c["timeouts"] == 0 and c["fp_mismatches"] == 0
    finally:
        run.close()


@pytest.mark.parametrize("P,Pp", [(1, 1), (2, 1), (4, 2), (8, 4), (8, 1), (3, 3)])
@pytest.mark.parametrize("fused", [True, False])
def test_parity_qgz(P, Pp, fused):
    """f1 qgZ: INT4 blockwise-quantized gradient all-to-all + fixed-order reduction, bit-exact
    vs the oracle's qgz_reduce_scatter (same fp32 rounding decisions for every code)."""
    run = ParityRun(NUMELS, P, Pp, qgz=True, fused=fused, verify="fingerprint")
    try:
        for _ in range(3):
            _check_step(run, run.step())
        assert run.counters()["timeouts"] == 0
    finally:
        run.close()


@pytest.mark.parametrize("P,Pp", [(1, 1), (2, 1), (4, 2), (8, 4), (8, 8), (3, 1)])
@pytest.mark.parametrize("fused", [True, False])
def test_parity_bf16_grads(P, Pp, fused):
    """f4: bf16 gradient slots, exact widening, fp32 fixed-order reduction: bit-exact."""
    run = ParityRun(NUMELS, P, Pp, grad_dtype="bf16", fused=fused, verify="fingerprint")
    try:
        for _ in range(3):
            _check_step(run, run.step())
        assert run.counters()["timeouts"] == 0
    finally:
        run.close()


@pytest.mark.parametrize("P,Pp", [(1, 1), (2, 1), (4, 2), (8, 4), (8, 8), (3, 1)])
@pytest.mark.parametrize("fused", [True, False])
def test_parity_qwz(P, Pp, fused):
    """f2 qwZ: INT8 blockwise weights in the forward gather, dequantized into the full
    buffer and the secondary: bit-exact vs the oracle (same fp32 decisions)."""
    run = ParityRun(NUMELS, P, Pp, qwz=True, fused=fused, verify="fingerprint")
    try:
        for _ in range(3):
            _check_step(run, run.step())
        c = run.counters()
        assert c["timeouts"] == 0 and c["fp_mismatches"] == 0
    finally:
        run.close()


def test_parity_qwz_fp32_params_and_qgz():
    """qwZ with fp32 parameters, combined with qgZ gradients (the paper's Table 2 runs qgZ)."""
    run = ParityRun(O.toy_layer_numels(), 4, 2, dtype="f32", qwz=True, qgz=True, fused=True, verify="fingerprint")
    try:
        for _ in range(2):
            _check_step(run, run.step())
    finally:
        run.close()


@pytest.mark.parametrize("P,Pp", [(1, 1), (4, 2), (8, 4)])
def test_parity_paper_order(P, Pp):
    """ORDER_PAPER (the paper's own host-side wait after a separate MemcpyD2D) is correct:
    same bits as the oracle's fixed ordering, 0 mismatches."""
    run = ParityRun(NUMELS, P, Pp, order="paper", verify="exact", fused=True)
    try:
        for _ in range(3):
            _check_step(run, run.step())
        c = run.counters()
        assert c["mismatches"] == 0 and c["timeouts"] == 0
    finally:
        run.close()


@pytest.mark.parametrize("P", [1, 2, 4, 8])
def test_secondary_aliased_when_node_is_the_world(P):
    """P' == P: secondary == primary, so the library stores no second copy —
    the secondary buffer IS the primary — the forward gather writes no secondary and the
    backward gather (reading the node's primaries) still returns W_t bitwise, with the
    optimizer ordered after it (E7).  EXACT verification re-reads the owners' primaries."""
    from paper_2407_01614_b200 import hpz as H
    run = ParityRun(NUMELS, P, P, fused=True, verify="exact", copy_engine="ldg")
    try:
        for rc in run.w.ranks:
            for i in range(len(NUMELS)):
                assert H.hpz_buffer(rc.ctx, i, "secondary") == (H.hpz_buffer(rc.ctx, i, "primary")[0],
                                                                 run.w.ranks[0].infos[i].shard)
        for _ in range(3):
            _check_step(run, run.step())
        c = run.counters()
        assert c["mismatches"] == 0 and c["nan_reads"] == 0 and c["timeouts"] == 0
    finally:
        run.close()


def test_parity_fused_off_order():
    run = ParityRun(NUMELS, 4, 2, order="off", fused=True)
    try:
        for _ in range(2):
            _check_step(run, run.step())
    finally:
        run.close()


@pytest.mark.parametrize("P,Pp", [(8, 4), (4, 2)])
def test_parity_off_equals_fixed(P, Pp):
    """ORDER_OFF (plain ZeRO-3 backward over P) gives the same bits (PAPER.md:207 / SPEC.md:352)."""
    run = ParityRun(NUMELS, P, Pp, order="off")
    try:
        for _ in range(2):
            _check_step(run, run.step())
        assert run.counters()["mismatches"] == 0
    finally:
        run.close()


@pytest.mark.parametrize("engine", ["ldg", "tma"])
def test_parity_fp32_params_toy_shapes(engine):
    """Config C1 shapes with fp32 parameters (primary == master copy)."""
    run = ParityRun(O.toy_layer_numels(), 8, 4, dtype="f32", copy_engine=engine, fused=engine == "tma")
    try:
        for _ in range(2):
            _check_step(run, run.step())
    finally:
        run.close()


def test_parity_dyadic_rs_closed_form():
    """Dyadic gradients: the GPU reduce-scatter equals the exact rational mean."""
    run = ParityRun([40_000], 8, 2, grad_kind="dyadic", verify="fingerprint")
    try:
        rec = run.step()
        _check_step(run, rec)
    finally:
        run.close()


def test_parity_shared_grad_slots():
    """Fewer gradient slots than layers: the E6 wait orders slot reuse."""
    run = ParityRun(NUMELS, 4, 2, n_grad_slots=2, verify="fingerprint")
    try:
        for _ in range(2):
            _check_step(run, run.step())
    finally:
        run.close()


def test_synth_generator_matches_host():
    """The device twin of synth/inputs.py produces the same fp32 bits."""
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import EmulatedWorld, buffer_view
    n = 123_457
    w = EmulatedWorld([n], 2, 1)
    try:
        s = torch.cuda.current_stream()
        for rc in w.ranks:
            H.hpz_synth_master(rc.ctx, 0, S.stream_key(S.SEED_PARAMS, 0, 0, 0), S.PARAM_SCALE, s)
            H.hpz_synth_grads(rc.ctx, 0, S.stream_key(S.SEED_GRADS, 0, 5, rc.rank), S.GRAD_SCALE, 0, s)
        torch.cuda.synchronize()
        full = S.layer_params(0, n, w.ranks[0].infos[0].numel_pad)
        for rc in w.ranks:
            info = rc.infos[0]
            m = buffer_view(rc, 0, "master", "f32").cpu().numpy()
            assert np.array_equal(m.view(np.uint32), full[rc.rank * info.shard:(rc.rank + 1) * info.shard].view(np.uint32))
            g = buffer_view(rc, 0, "grad_slot", "f32").cpu().numpy()
            ref = S.layer_grads(0, 5, rc.rank, n, info.numel_pad)
            assert np.array_equal(g.view(np.uint32), ref.view(np.uint32))
            # bf16 primary = RNE(master)
            p = bits_np(buffer_view(rc, 0, "primary", "bf16"), "bf16")
            assert np.array_equal(p, O.bf16_rne(m))
    finally:
        w.close()


def test_stock_ordering_shows_stale_reads():
    """Negative control (Table 1 ×): stock ordering with a delayed,
    poisoned side-stream secondary copy makes backward gathers read stale or NaN
    weights; the exact detector counts them (> 0; the count itself is a hardware race)."""
    from paper_2407_01614_b200 import hpz as H
    run = ParityRun(NUMELS, 8, 4, order="stock", verify="exact")
    try:
        for rc in run.w.ranks:
            H.hpz_set_order(rc.ctx, "stock", stock_delay_us=2000, stock_poison=True)
        for _ in range(3):
            run.step()
        c = run.counters()
        assert c["mismatches"] > 0
        assert c["timeouts"] == 0
    finally:
        run.close()


def test_api_errors():
    from paper_2407_01614_b200 import hpz as H
    with pytest.raises(H.HpzError) as e:
        H.hpz_init(8, 3, 0, 0)
    assert e.value.code == H.HPZ_EINVAL
    ctx = H.hpz_init(2, 2, 0, 0)
    try:
        with pytest.raises(H.HpzError) as e:
            H.hpz_fwd_gather(ctx, 0, 0)
        assert e.value.code == H.HPZ_ESTATE
        H.hpz_register_flat_params(ctx, [1000])
        with pytest.raises(H.HpzError) as e:
            H.hpz_register_flat_params(ctx, [1000])
        assert e.value.code == H.HPZ_ESTATE
    finally:
        H.hpz_finalize(ctx)
    from paper_2407_01614_b200.world import EmulatedWorld
    w = EmulatedWorld([5000], 2, 2)
    try:
        buf = torch.empty(w.ranks[0].infos[0].numel_pad, dtype=torch.bfloat16, device="cuda")
        with pytest.raises(H.HpzError) as e:   # backward before forward
            H.hpz_bwd_gather(w.ranks[0].ctx, 0, buf.data_ptr())
        assert e.value.code == H.HPZ_ESTATE
        with pytest.raises(H.HpzError) as e:   # misaligned output
            H.hpz_fwd_gather(w.ranks[0].ctx, 0, buf.data_ptr() + 2)
        assert e.value.code == H.HPZ_EINVAL
        with pytest.raises(H.HpzError) as e:   # step before reduce-scatter
            H.hpz_step(w.ranks[0].ctx, 0, H.make_adam())
        assert e.value.code == H.HPZ_ESTATE
    finally:
        w.close()


def test_missing_peer_times_out_instead_of_hanging():
    """Failure detection: a backward gather whose node peer never released its secondary
    (the peer skipped its forward) waits at most the timeout, records it, and the next
    call on that context returns HPZ_ETIMEOUT — the GPU is never hung."""
    import time
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import EmulatedWorld
    w = EmulatedWorld([50_000], 4, 2, timeout_s=1.0)
    try:
        s = torch.cuda.current_stream()
        w0 = torch.from_numpy(S.layer_params(0, 50_000)).cuda()
        for rc in w.ranks:
            H.hpz_load_master(rc.ctx, 0, w0.data_ptr(), s)
        buf = torch.empty(w.ranks[0].infos[0].numel_pad, dtype=torch.bfloat16, device="cuda")
        r0 = w.ranks[0].ctx
        H.hpz_fwd_gather(r0, 0, buf.data_ptr(), s)       # rank 1 never runs its forward
        t0 = time.time()
        H.hpz_bwd_gather(r0, 0, buf.data_ptr(), s)       # waits for rank 1's SEC_READY
        torch.cuda.synchronize()
        assert time.time() - t0 < 30
        c = H.hpz_counters(r0)
        assert c["timeouts"] >= 1
        with pytest.raises(H.HpzError) as e:
            H.hpz_grad_buffer(r0, 0, s)
        assert e.value.code == H.HPZ_ETIMEOUT
        # the error names the edge that never arrived (first timed-out flag, decoded)
        assert "SEC_READY (E3) of layer 0 from rank 1" in str(e.value), str(e.value)
    finally:
        w.close()


@pytest.mark.parametrize("P", [1, 2])
def test_qgz_quantizer_ties_and_edges(P):
    """The division-free quantizer (quant_code) must reproduce round-half-even of the IEEE
    quotient exactly, including exact ties, near-ties, constant blocks, tiny/huge scales."""
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import EmulatedWorld, buffer_view, run_step
    rng = np.random.default_rng(3)
    n = 64 * 64
    blocks = []
    for b in range(64):
        kind = b % 8
        base = np.zeros(64, np.float32)
        if kind == 0:   # exact ties: mn 0, mx 15 -> scale 1, values k + 0.5
            base = (np.arange(64) % 16).astype(np.float32) + np.float32(0.5) * (np.arange(64) % 2)
            base[0], base[1] = 0.0, 15.0
        elif kind == 1:  # scaled ties (scale 2^-10)
            base = ((np.arange(64) % 31) * 0.5).astype(np.float32) * np.float32(2 ** -10)
            base[0], base[1] = 0.0, 15.0 * 2 ** -10
        elif kind == 2:  # near ties: one ulp either side of k + 0.5 (scale 1)
            k = (np.arange(64) % 15).astype(np.float32) + np.float32(0.5)
            base = np.where(np.arange(64) % 2 == 0, np.nextafter(k, np.float32(0)), np.nextafter(k, np.float32(20)))
            base = base.astype(np.float32)
            base[0], base[1] = 0.0, 15.0
        elif kind == 3:  # constant block
            base[:] = np.float32(0.3)
        elif kind == 4:  # tiny dynamic range
            base = (np.float32(1.0) + rng.integers(0, 16, 64).astype(np.float32) * np.float32(2 ** -23)).astype(np.float32)
        elif kind == 5:  # huge values
            base = (rng.standard_normal(64) * 1e30).astype(np.float32)
        else:
            base = (rng.standard_normal(64) * 10 ** rng.uniform(-8, 3)).astype(np.float32)
        blocks.append(base)
    g_full = np.concatenate(blocks).astype(np.float32)
    from oracle import hpz_oracle as O
    w = EmulatedWorld([n], P, 1, qgz=True, timeout_s=10.0)
    try:
        s = torch.cuda.current_stream()
        w0 = torch.zeros(n, dtype=torch.float32, device="cuda")
        for rc in w.ranks:
            H.hpz_load_master(rc.ctx, 0, w0.data_ptr(), s)
        out = [torch.empty(rc.infos[0].numel_pad, dtype=torch.bfloat16, device="cuda") for rc in w.ranks]
        gs = [torch.from_numpy(g_full * np.float32(r + 1)).cuda() for r in range(P)]

        def grad_fn(rc, i):
            H.hpz_grad_upload(rc.ctx, i, gs[rc.rank].data_ptr(), n, s)

        run_step(w.ranks, [lambda i, r=r: out[r].data_ptr() for r in range(P)],
                 [lambda i, r=r: out[r].data_ptr() for r in range(P)], H.make_adam(), stream=s,
                 grad_fn=grad_fn, emulated=True)
        torch.cuda.synchronize()
        lay = O.LayerLayout(n, P, 1, 256)
        G = [O.pad_full(g_full * np.float32(r + 1), lay) for r in range(P)]
        for rc in w.ranks:
            got = buffer_view(rc, 0, "grad_shard", "f32").cpu().numpy()
            ref = O.qgz_reduce_scatter(G, lay, rc.rank)
            assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))
    finally:
        w.close()


def test_checkpoint_resume_is_bit_identical():
    """Checkpoint/resume: 2 steps, save (master, m, v, Adam count), fresh world,
    load, 1 step == 3 uninterrupted steps, bit for bit (and == the oracle)."""
    from paper_2407_01614_b200.world import load_checkpoint, save_checkpoint
    ref = ParityRun(NUMELS, 4, 2, fused=True, verify="fingerprint")
    try:
        for _ in range(3):
            rec = ref.step()
        _check_step(ref, rec)
        want = [[buffer_view_f32(rc, i) for i in range(len(NUMELS))] for rc in ref.w.ranks]
    finally:
        ref.close()
    a = ParityRun(NUMELS, 4, 2, fused=True, verify="fingerprint")
    try:
        for _ in range(2):
            a.step()
        ckpts = [save_checkpoint(rc, 2) for rc in a.w.ranks]
    finally:
        a.close()
    b = ParityRun(NUMELS, 4, 2, fused=True, verify="fingerprint", load_initial=False)
    try:
        for rc, ck in zip(b.w.ranks, ckpts):
            load_checkpoint(rc, ck, b.stream)
        b.t = 2                       # the gradient generator continues at step 2
        b.step(run_oracle=False)
        for r, rc in enumerate(b.w.ranks):
            for i in range(len(NUMELS)):
                assert np.array_equal(buffer_view_f32(rc, i), want[r][i])
    finally:
        b.close()


def buffer_view_f32(rc, i):
    from paper_2407_01614_b200.world import buffer_view
    return buffer_view(rc, i, "master", "f32").cpu().numpy().view(np.uint32).copy()


def test_order_switch_between_steps():
    """hpz_set_order may change between steps (all ranks alike): fixed -> off -> paper ->
    fixed trains exactly like fixed throughout (all orders compute the same values)."""
    from paper_2407_01614_b200 import hpz as H
    run = ParityRun(NUMELS, 4, 2, fused=True, verify="fingerprint")
    try:
        for order in ("fixed", "off", "paper", "fixed"):
            for rc in run.w.ranks:
                H.hpz_set_order(rc.ctx, order)
            # an OFF step writes no secondary (plain ZeRO-3): its content is step t-1's
            _check_step(run, run.step(), check_secondary=order != "off")
        assert run.counters()["timeouts"] == 0
    finally:
        run.close()


def test_paper_order_with_one_reused_full_buffer():
    """ORDER_PAPER's MemcpyD2D reads the caller's full buffer on a side
    stream.  A caller that reuses one full buffer for every layer (the bench; a prefetch
    ring) must never let the next layer's gather overwrite it before the copy has read it
    (regression: the secondary received the next layer's parameters and the backward
    gather read them).  A 3 ms delay before each copy widens the window; EXACT verification
    compares every backward-gathered element with the owners' primaries."""
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import EmulatedWorld, buffer_view, run_step
    numels = [300_007, 250_000, 65_536]
    P, Pp = 4, 2
    w = EmulatedWorld(numels, P, Pp, timeout_s=10.0)
    o = O.HpzOracle(numels, P, Pp, align=256, order="fixed")
    try:
        s = torch.cuda.current_stream()
        for rc in w.ranks:
            H.hpz_set_order(rc.ctx, "paper", stock_delay_us=3000)
            H.hpz_set_verify(rc.ctx, "exact")
        for i, n in enumerate(numels):
            w0 = torch.from_numpy(S.layer_params(i, n)).cuda()
            for rc in w.ranks:
                H.hpz_load_master(rc.ctx, i, w0.data_ptr(), s)
        nmax = max(x.numel_pad for x in w.ranks[0].infos)
        fwd = [torch.empty(nmax, dtype=torch.bfloat16, device="cuda") for _ in range(P)]   # one per rank, all layers
        bwd = [torch.empty(nmax, dtype=torch.bfloat16, device="cuda") for _ in range(P)]
        keep = []
        t_box = [0]

        def grad_fn(rc, i):
            g = torch.from_numpy(S.layer_grads(i, t_box[0], rc.rank, numels[i])).cuda()
            keep.append(g)
            H.hpz_grad_upload(rc.ctx, i, g.data_ptr(), numels[i], s)

        adam = H.make_adam()
        for t in range(3):
            t_box[0] = t
            run_step(w.ranks, [lambda i, r=r: fwd[r].data_ptr() for r in range(P)],
                     [lambda i, r=r: bwd[r].data_ptr() for r in range(P)], adam, stream=s, grad_fn=grad_fn,
                     emulated=True, fused=True)
            torch.cuda.synchronize()
            o.step()
        tot = {}
        for rc in w.ranks:
            for k, v in H.hpz_counters(rc.ctx).items():
                tot[k] = tot.get(k, 0) + v
        assert tot["mismatches"] == 0 and tot["nan_reads"] == 0 and tot["timeouts"] == 0, tot
        for i in range(len(numels)):
            for rc in w.ranks:
                got = buffer_view(rc, i, "master", "f32").cpu().numpy()
                assert np.array_equal(got.view(np.uint32), o.state[i][rc.rank].master.view(np.uint32)), (i, rc.rank)
    finally:
        w.close()


# ---------------------------------------------------------------- a7: owner-emitted fingerprints
def test_forward_fingerprint_checked_against_owners():
    """FINGERPRINT mode compares every forward gather with the checksum its owners emitted
    when they wrote the primaries (init, then every Adam): all checked, none differ."""
    run = ParityRun(NUMELS, 4, 2, fused=True, verify="fingerprint")
    try:
        for _ in range(3):
            _check_step(run, run.step())
        c = run.counters()
        assert c["fp_fwd_checked"] == 3 * len(NUMELS) * 4 and c["fp_fwd_mismatches"] == 0, c
        assert c["fp_checked"] == 3 * len(NUMELS) * 4 and c["fp_mismatches"] == 0, c
    finally:
        run.close()


def test_forward_fingerprint_qwz_and_unfused():
    """Same with qwZ (the quantizer emits the dequantized words' checksum) and with the
    unfused Adam kernel."""
    for kw in (dict(qwz=True, fused=True), dict(fused=False), dict(fused=False, copy_engine="ldg")):
        run = ParityRun(NUMELS, 4, 2, verify="fingerprint", **kw)
        try:
            for _ in range(2):
                _check_step(run, run.step())
            c = run.counters()
            assert c["fp_fwd_checked"] == 2 * len(NUMELS) * 4 and c["fp_fwd_mismatches"] == 0, (kw, c)
        finally:
            run.close()


def _sleep_ms(ms, stream):
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(ms * 2.0e6))     # ~2 GHz SM clock


@pytest.mark.parametrize("fault", [0, 1])
def test_fingerprint_catches_forward_read_before_adam(fault):
    """E1 (PRIMARY_READY) removed on purpose (HPZ_FAULT_SKIP_E1): the owner's Adam of step 0
    is held back on a side stream while the forward gathers of step 1 run — they read the
    pre-step primary and the forward-vs-owner fingerprint fires.  With the edge in place
    (fault 0) the same schedule waits and reads W_1: no mismatch.  Grids are capped so the
    waiting kernels never fill the GPU (B200_PROFILING.md)."""
    from paper_2407_01614_b200 import hpz as H
    numels = [300_007, 65_536]
    run = ParityRun(numels, 2, 1, fused=True, verify="fingerprint")
    try:
        for rc in run.w.ranks:
            H.hpz_set_option(rc.ctx, "max_ctas", 32)
        _check_step(run, run.step())
        run.counters()                                   # reset
        main, side = run.stream, torch.cuda.Stream()
        bufs = run.fwd
        for rc in run.w.ranks:
            H.hpz_set_option(rc.ctx, "fault", H.FAULT_SKIP_E1 if fault else 0)
        run._keep = []
        L = len(numels)
        for i in range(L):
            for rc in run.w.ranks:
                H.hpz_fwd_gather(rc.ctx, i, bufs[rc.rank][i].data_ptr(), main)
        for i in reversed(range(L)):
            for rc in run.w.ranks:
                H.hpz_bwd_gather(rc.ctx, i, run.bwd[rc.rank][i].data_ptr(), main)
            for rc in run.w.ranks:
                run.grad_fn(rc, i)
                H.hpz_grads_ready(rc.ctx, i, main)
        side.wait_stream(main)
        _sleep_ms(50, side)
        for i in reversed(range(L)):
            H.hpz_reduce_scatter_adam(run.w.ranks[0].ctx, i, run.adam, side)   # owner 0: late
            H.hpz_reduce_scatter_adam(run.w.ranks[1].ctx, i, run.adam, main)
        for i in range(L):                                                   # step 1 forward
            for rc in run.w.ranks:
                H.hpz_fwd_gather(rc.ctx, i, bufs[rc.rank][i].data_ptr(), main)
        torch.cuda.synchronize()
        c = run.counters()
        assert c["timeouts"] == 0, c
        if fault:
            assert c["fp_fwd_mismatches"] > 0, c
        else:
            assert c["fp_fwd_mismatches"] == 0 and c["fp_fwd_checked"] == 2 * L * 2, c
    finally:
        run.close()


@pytest.mark.parametrize("fault", [0, 2])
def test_fingerprint_catches_adam_overwriting_a_read_primary(fault):
    """E2 (FWD_DONE) removed on purpose (HPZ_FAULT_SKIP_E2): rank 1 publishes its step-1
    gradients early (hpz_grads_ready) and its forward gathers of step 1 lag on another stream,
    so nothing but E2 keeps owner 0's Adam from overwriting its primary with W_2 while rank 1
    still has to read W_1.  Without E2 rank 1 gathers the wrong version and its forward
    fingerprint differs from the owners'; with E2 (fault 0) the same schedule is safe."""
    from paper_2407_01614_b200 import hpz as H
    numels = [300_007, 65_536]
    run = ParityRun(numels, 2, 1, fused=True, verify="fingerprint")
    try:
        for rc in run.w.ranks:
            H.hpz_set_option(rc.ctx, "max_ctas", 32)
        _check_step(run, run.step())
        run.counters()                                   # reset
        main, s1, sdelay = run.stream, torch.cuda.Stream(), torch.cuda.Stream()
        r0, r1 = run.w.ranks
        H.hpz_set_option(r0.ctx, "fault", fault)
        L = len(numels)
        gs = {(rc.rank, i): torch.from_numpy(S.layer_grads(i, run.t, rc.rank, lay.numel)).cuda()
              for rc in run.w.ranks for i, lay in enumerate(run.o.layouts)}
        torch.cuda.synchronize()
        for i in reversed(range(L)):                     # rank 1: gradients first (early E5)
            H.hpz_grad_upload(r1.ctx, i, gs[(1, i)].data_ptr(), numels[i], s1)
            H.hpz_grads_ready(r1.ctx, i, s1)
        _sleep_ms(50, sdelay)
        for i in range(L):
            H.hpz_fwd_gather(r0.ctx, i, run.fwd[0][i].data_ptr(), main)
            H.hpz_fwd_gather(r1.ctx, i, run.fwd[1][i].data_ptr(), sdelay)     # rank 1 lags
        for i in reversed(range(L)):
            H.hpz_bwd_gather(r0.ctx, i, run.bwd[0][i].data_ptr(), main)
            H.hpz_bwd_gather(r1.ctx, i, run.bwd[1][i].data_ptr(), sdelay)
            H.hpz_grad_upload(r0.ctx, i, gs[(0, i)].data_ptr(), numels[i], main)
            H.hpz_grads_ready(r0.ctx, i, main)
            H.hpz_reduce_scatter_adam(r0.ctx, i, run.adam, main)
            H.hpz_reduce_scatter_adam(r1.ctx, i, run.adam, sdelay)
        torch.cuda.synchronize()
        c1 = H.hpz_counters(r1.ctx)
        c0 = H.hpz_counters(r0.ctx)
        assert c0["timeouts"] == 0 and c1["timeouts"] == 0
        if fault:
            assert c1["fp_fwd_mismatches"] > 0, c1
        else:
            assert c1["fp_fwd_mismatches"] == 0 and c0["fp_fwd_mismatches"] == 0, (c0, c1)
            assert c1["fp_fwd_checked"] == L and c0["fp_fwd_checked"] == L, (c0, c1)
    finally:
        run.close()


# ---------------------------------------------------------------- device epochs + CUDA graphs
@pytest.mark.parametrize("P,Pp,kw", [(4, 2, {}), (2, 2, {}), (4, 2, {"qgz": True}), (2, 1, {"grad_dtype": "bf16"}),
                                     (1, 1, {})])
def test_captured_step_replays_bit_exact(P, Pp, kw):
    """with device-side epochs a whole training step (every rank's gathers,
    gradient uploads, fused RS+Adam) is captured ONCE in a CUDA graph and replayed; each
    replay is a new step — fresh flag epochs and Adam bias corrections from the device
    counter — and matches the oracle bit for bit over 3 replays, then eager steps resume."""
    from paper_2407_01614_b200 import hpz as H
    run = ParityRun(NUMELS, P, Pp, fused=True, verify="fingerprint", **kw)
    try:
        for rc in run.w.ranks:
            H.hpz_set_option(rc.ctx, "device_epoch", 1)
        _check_step(run, run.step())                 # eager step 0 in device-epoch mode
        L = len(NUMELS)
        gdt = torch.bfloat16 if run.grad_dtype == "bf16" else torch.float32
        gstatic = [[torch.zeros(run.o.layouts[i].numel, dtype=gdt, device="cuda") for i in range(L)]
                   for _ in range(P)]

        def fill(t):
            for r in range(P):
                for i, lay in enumerate(run.o.layouts):
                    g = torch.from_numpy(S.layer_grads(i, t, r, lay.numel, kind=run.grad_kind)).cuda()
                    gstatic[r][i].copy_(g.to(gdt))
            torch.cuda.synchronize()

        def grad_fn(rc, i):
            H.hpz_grad_upload(rc.ctx, i, gstatic[rc.rank][i].data_ptr(), run.o.layouts[i].numel,
                              torch.cuda.current_stream())

        from paper_2407_01614_b200.world import run_step
        graph = torch.cuda.CUDAGraph()
        fill(1)
        with torch.cuda.graph(graph):
            run_step(run.w.ranks, [lambda i, r=r: run.fwd[r][i].data_ptr() for r in range(P)],
                     [lambda i, r=r: run.bwd[r][i].data_ptr() for r in range(P)], run.adam,
                     stream=torch.cuda.current_stream(), grad_fn=grad_fn, emulated=True, fused=True)
        for k in range(3):                          # replays = steps 1, 2, 3
            fill(1 + k)
            graph.replay()
            torch.cuda.synchronize()
            run.t = 1 + k
            rec = run.o.step()
            run.t = 2 + k
            _check_step(run, rec)
        for rc in run.w.ranks:
            H.hpz_resync_step(rc.ctx)
            assert H.hpz_current_step(rc.ctx) == 4
        _check_step(run, run.step())                 # eager step 4
        c = run.counters()
        assert c["timeouts"] == 0 and c["fp_mismatches"] == 0 and c["fp_fwd_mismatches"] == 0, c
        assert c["fp_checked"] == 5 * L * P and c["fp_fwd_checked"] == 5 * L * P, c
    finally:
        run.close()


def test_device_epoch_rejects_uncapturable_orders():
    from paper_2407_01614_b200 import hpz as H
    run = ParityRun(NUMELS, 2, 1, fused=True)
    try:
        for rc in run.w.ranks:
            H.hpz_set_option(rc.ctx, "device_epoch", 1)
            H.hpz_set_order(rc.ctx, "paper")
        with pytest.raises(H.HpzError) as e:
            H.hpz_fwd_gather(run.w.ranks[0].ctx, 0, run.fwd[0][0].data_ptr(), run.stream)
        assert e.value.code == H.HPZ_ESTATE
    finally:
        run.close()


def test_checkpoint_rejects_a_different_shard_layout():
    """A checkpoint written under another align_elems (another padding, so another shard
    length) is rejected before any raw copy (hpz_load_state copies `shard` elements)."""
    from paper_2407_01614_b200.world import load_checkpoint, save_checkpoint
    a = ParityRun([100_003], 4, 2, fused=True, verify="none", align=256)
    try:
        a.step()
        ck = save_checkpoint(a.w.ranks[1], 1)
    finally:
        a.close()
    b = ParityRun([100_003], 4, 2, fused=True, verify="none", align=8, load_initial=False)
    try:
        assert b.w.ranks[1].infos[0].shard != ck["shards"][0]
        with pytest.raises(ValueError):
            load_checkpoint(b.w.ranks[1], ck, b.stream)
    finally:
        b.close()


# ---------------------------------------------------------------- ranks on concurrent streams
@pytest.mark.parametrize("P,Pp,kw", [(4, 2, {}), (2, 2, {}), (8, 4, {"qgz": True}), (4, 1, {"grad_dtype": "bf16"}),
                                     (4, 2, {"device_epoch": True})])
def test_emulated_ranks_on_concurrent_streams(P, Pp, kw):
    """Single-GPU emulation with one stream PER RANK: each rank's calls go to its own stream,
    so the ranks' kernels run concurrently and every cross-rank flag wait (E1-E7) is a real
    race between running kernels, not satisfied by stream order as in the one-stream
    emulation.  Two rules keep mutually-waiting kernels on one GPU deadlock-free (a
    multi-process world with one GPU per rank needs neither): calls are submitted in SPMD
    phase order across ranks (every kernel is submitted after the kernels whose flags it
    waits for — the driver may serialize several streams in one hardware queue, measured: a
    rank-by-rank submission deadlocked on E3 with 36-CTA grids), and grids are capped so all
    ranks' waiting kernels fit on the GPU at once.  3 steps, bit-exact vs the oracle, all
    fingerprints checked."""
    from paper_2407_01614_b200 import hpz as H
    kw = dict(kw)
    dev_epoch = kw.pop("device_epoch", False)
    run = ParityRun(NUMELS, P, Pp, fused=True, verify="fingerprint", **kw)
    try:
        streams = [torch.cuda.Stream() for _ in range(P)]
        for rc in run.w.ranks:
            H.hpz_set_option(rc.ctx, "max_ctas", 144 // P)
            if dev_epoch:
                H.hpz_set_option(rc.ctx, "device_epoch", 1)
        L = len(NUMELS)
        ranks = run.w.ranks
        for t in range(3):
            grads = {(r, i): torch.from_numpy(np.ascontiguousarray(run.grads(i, t, r)[:run.o.layouts[i].numel])).cuda()
                     for r in range(P) for i in range(L)}
            if run.grad_dtype == "bf16":
                grads = {k: v.to(torch.bfloat16) for k, v in grads.items()}
            torch.cuda.synchronize()
            for i in range(L):
                for rc in ranks:
                    H.hpz_fwd_gather(rc.ctx, i, run.fwd[rc.rank][i].data_ptr(), streams[rc.rank])
            for i in reversed(range(L)):
                for rc in ranks:
                    H.hpz_bwd_gather(rc.ctx, i, run.bwd[rc.rank][i].data_ptr(), streams[rc.rank])
                for rc in ranks:
                    H.hpz_grad_upload(rc.ctx, i, grads[(rc.rank, i)].data_ptr(), run.o.layouts[i].numel,
                                      streams[rc.rank])
                    H.hpz_grads_ready(rc.ctx, i, streams[rc.rank])
                for rc in ranks:
                    H.hpz_reduce_scatter_adam(rc.ctx, i, run.adam, streams[rc.rank])
            torch.cuda.synchronize()
            rec = run.o.step()
            run.t = t + 1
            _check_step(run, rec)
        c = run.counters()
        assert c["timeouts"] == 0 and c["fp_mismatches"] == 0 and c["fp_fwd_mismatches"] == 0, c
        assert c["fp_checked"] == 3 * L * P and c["fp_fwd_checked"] == 3 * L * P, c
    finally:
        run.close()
