"""Stock ZeRO++ ordering under Algorithm 1's own prefetch schedule (PAPER.md:84-118,
130-137): which backward gathers race with their secondary copy.

The oracle's "realistic" schedule (oracle.realistic_racing_layers) predicts, from the
program order alone, the layers whose backward AllGather(L_i, P') is enqueued before the
copy that fills L_i's secondary: the last ceil(d/2) layers at prefetch depth d (the
forward->backward turnaround of Fig. 1).  Here the same schedule runs on the GPU: the
gathers on a communication stream, each into a ring of d+1 full buffers (a buffer is reused
only after the compute that read it — ZeRO-3's repartition), the compute of
each module as a fixed-length kernel on a compute stream, and the stock secondary copy
issued by the caller after each forward (HPZ_OPT_COPY_BY_CALLER, hpz_secondary_copy, as
Alg. 1 does).  The stock backward gather waits for nothing, so it reads a stale secondary
exactly on the predicted layers; every other layer's copy landed first.  With the fix
(ORDER_FIXED) the same schedule reads W_t everywhere.  The mismatch COUNTS are a hardware
race (R25); the test asserts the set of layers that mismatch.
"""
import numpy as np
import pytest
import torch

from oracle import hpz_oracle as O
from synth import inputs as S

from .gpu_util import bits_np, gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a GPU")]

COMPUTE_MS = 4.0      # each module's compute (a spin kernel on the compute stream)
COPY_DELAY_US = 1000  # the stock copy's lag behind its forward (well under one module)


def _sleep(ms, stream):
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(ms * 2.0e6))


def _run_schedule(order, depth, steps=2, P=4, Pp=2, numels=(300_007, 65_536, 250_000, 4_099, 120_000)):
    from paper_2407_01614_b200 import hpz as H
    from paper_2407_01614_b200.world import EmulatedWorld
    numels = list(numels)
    N = len(numels)
    w = EmulatedWorld(numels, P, Pp, timeout_s=10.0)
    o = O.HpzOracle(numels, P, Pp, order="fixed")
    comm, comp = torch.cuda.Stream(), torch.cuda.Stream()
    try:
        for rc in w.ranks:
            H.hpz_set_order(rc.ctx, order, stock_delay_us=COPY_DELAY_US if order == "stock" else 0)
            H.hpz_set_option(rc.ctx, "copy_by_caller", int(order == "stock"))
            H.hpz_set_option(rc.ctx, "max_ctas", 32)
        for i, n in enumerate(numels):
            w0 = torch.from_numpy(S.layer_params(i, n)).cuda()
            for rc in w.ranks:
                H.hpz_load_master(rc.ctx, i, w0.data_ptr())
        torch.cuda.synchronize()
        R = depth + 1
        npad = max(x.numel_pad for x in w.ranks[0].infos)
        ring = [[torch.zeros(npad, dtype=torch.bfloat16, device="cuda") for _ in range(R)] for _ in range(P)]
        snap = [[torch.zeros(x.numel_pad, dtype=torch.bfloat16, device="cuda") for x in w.ranks[0].infos]
                for _ in range(P)]
        adam = H.make_adam()
        modules = [("fwd", i) for i in range(N)] + [("bwd", i) for i in reversed(range(N))]
        per_step = []
        for t in range(steps):
            grads = [[torch.from_numpy(S.layer_grads(i, t, r, numels[i])).cuda() for i in range(N)] for r in range(P)]
            torch.cuda.synchronize()
            ready = [torch.cuda.Event() for _ in range(R)]
            free = [None] * R
            enq, k = {}, [0]

            def gather(m):
                slot = k[0] % R
                k[0] += 1
                if free[slot] is not None:
                    comm.wait_event(free[slot])          # repartition: the buffer's reader is done
                fn = H.hpz_fwd_gather if m[0] == "fwd" else H.hpz_bwd_gather
                for rc in w.ranks:
                    fn(rc.ctx, m[1], ring[rc.rank][slot].data_ptr(), comm)
                ready[slot].record(comm)
                enq[m] = slot

            for pos, m in enumerate(modules):
                if m not in enq:
                    gather(m)                            # Ensure AllGather(L_i) finished
                for nxt in modules[pos + 1:pos + 1 + depth]:
                    if nxt not in enq:
                        gather(nxt)                      # PrefetchAllGather()
                slot = enq[m]
                comp.wait_event(ready[slot])
                _sleep(COMPUTE_MS, comp)                 # L_i.forward() / L_i.backward()
                i = m[1]
                if m[0] == "fwd":
                    if order == "stock":                 # L_i,second <- empty; async copy
                        for rc in w.ranks:
                            H.hpz_secondary_copy(rc.ctx, i, comp)
                else:
                    with torch.cuda.stream(comp):
                        for r in range(P):
                            snap[r][i].copy_(ring[r][slot][:snap[r][i].numel()])
                    for rc in w.ranks:
                        H.hpz_grad_upload(rc.ctx, i, grads[rc.rank][i].data_ptr(), numels[i], comp)
                    comm.wait_stream(comp)
                    for rc in w.ranks:
                        H.hpz_grads_ready(rc.ctx, i, comm)
                    for rc in w.ranks:
                        H.hpz_reduce_scatter_adam(rc.ctx, i, adam, comm)
                ev = torch.cuda.Event()
                ev.record(comp)
                free[slot] = ev
            torch.cuda.synchronize()
            rec = o.step()
            per_step.append([sum(int(np.count_nonzero(bits_np(snap[r][i], "bf16")[:numels[i]] !=
                                                       O.param_bits(rec.W[i], "bf16")[:numels[i]]))
                                 for r in range(P)) for i in range(N)])
            keep = grads   # noqa: F841  (uploads read them until the step is done)
        c = [H.hpz_counters(rc.ctx) for rc in w.ranks]
        assert all(x["timeouts"] == 0 for x in c)
        return per_step
    finally:
        w.close()


@pytest.mark.parametrize("depth", [1, 3])
def test_stock_races_exactly_the_predicted_layers(depth):
    numels = (300_007, 65_536, 250_000, 4_099, 120_000)
    racing = O.realistic_racing_layers(len(numels), depth)
    per_step = _run_schedule("stock", depth, numels=numels)
    for t, mism in enumerate(per_step):
        got = {i for i, m in enumerate(mism) if m > 0}
        assert got == racing, (t, mism, racing)


def test_fixed_order_same_schedule_reads_w_t():
    """The fix under the same prefetching schedule: E3 makes every backward gather wait for
    its secondary (written by the forward gather's fused store), so nothing is stale."""
    per_step = _run_schedule("fixed", 1)
    assert all(m == 0 for mism in per_step for m in mism), per_step
