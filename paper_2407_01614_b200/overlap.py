"""f3: Algorithm 1's PrefetchAllGather on B200 streams, around real compute.

Alg. 1 enqueues the AllGather of the next module(s) ahead of the one
being computed ("PrefetchAllGather"), forward over P and backward over P'.  Here the
gathers run on a communication stream, the model's GEMMs (cuBLAS through torch — the
plain library GEMMs the task allows) on the compute stream; CUDA events order the two
streams of ONE rank, and libhpz's device flags order the ranks.  The paper's fix needs
no host wait: the backward gather acquires SEC_READY on the device.

Two models (`model=`):
* "mlp": L layers, layer i holds one weight W_i (h x h, bf16); forward
  h_{i+1} = relu(h_i W_i^T) (no relu on the last), loss = mean((h_L - y)^2); backward
  dW_i = dY_i^T h_i written straight into the layer's bf16 gradient slot (f4),
  dh_i = dY_i W_i computed with the BACKWARD-gathered W_i.
* "transformer": L pre-norm decoder blocks (RMSNorm, causal multi-head self-attention
  through torch's fused SDPA, RMSNorm, GELU MLP; bf16 GEMMs on the tensor cores), one flat
  parameter buffer per block (`block_numel`).  The forward keeps only each block's input
  (activation checkpointing, as ZeRO-3 training of large models does); the backward
  recomputes block i from the BACKWARD-gathered parameters under autograd and copies the
  flat parameter gradient into the block's bf16 gradient slot.
In both, the backward math uses the backward-gathered weights — so a stale or poisoned
secondary (stock ordering) corrupts the gradients exactly as in the paper.
"""
from __future__ import annotations

import torch
import torch.nn.functional as F

from . import hpz as H
from .world import device_view


def block_numel(h: int, f: int) -> int:
    """Flat parameters of one decoder block: Wqkv (3h x h), Wo (h x h), W1 (f x h),
    W2 (h x f), RMSNorm gains g1, g2 (h each, applied as 1 + g)."""
    return 4 * h * h + 2 * h * f + 2 * h


def block_forward(flat: torch.Tensor, x: torch.Tensor, h: int, f: int, n_heads: int) -> torch.Tensor:
    """One pre-norm decoder block on x (B, S, h), parameters viewed from the flat buffer."""
    o = 0

    def take(n, shape):
        nonlocal o
        v = flat[o:o + n].view(*shape)
        o += n
        return v
    wqkv = take(3 * h * h, (3 * h, h))
    wo = take(h * h, (h, h))
    w1 = take(f * h, (f, h))
    w2 = take(h * f, (h, f))
    g1 = take(h, (h,))
    g2 = take(h, (h,))
    B, S, _ = x.shape
    d = h // n_heads

    def rms(t, g):
        tf = t.float()
        return (tf * torch.rsqrt(tf.pow(2).mean(-1, keepdim=True) + 1e-6)).to(t.dtype) * (1 + g)
    q, k, v = (rms(x, g1) @ wqkv.t()).view(B, S, 3, n_heads, d).permute(2, 0, 3, 1, 4)
    a = F.scaled_dot_product_attention(q, k, v, is_causal=True)
    x = x + a.transpose(1, 2).reshape(B, S, h) @ wo.t()
    return x + F.gelu(rms(x, g2) @ w1.t()) @ w2.t()


class GatherRing:
    """n full-parameter buffers reused round-robin; each has a 'ready' event (gather done,
    recorded on the comm stream) and a 'free' event (consumer done, compute stream)."""

    def __init__(self, n: int, numel_pad: int, dtype, device):
        self.bufs = [torch.empty(numel_pad, dtype=dtype, device=device) for _ in range(n)]
        self.ready = [torch.cuda.Event() for _ in range(n)]
        self.free = [None] * n
        self.n = n

    def slot(self, k: int) -> int:
        return k % self.n


class PrefetchTrainer:
    """One rank's training loop with prefetch depth `depth` (0 = gather on demand)."""

    def __init__(self, rc, h: int, L: int, tokens: int, depth: int = 1, n_bufs: int = 3,
                 comm_stream=None, compute_stream=None, lr: float = 1e-3, model: str = "mlp",
                 ffn: int | None = None, n_heads: int = 16, grad_dtype: str = "bf16"):
        self.rc, self.ctx, self.h, self.L, self.T = rc, rc.ctx, h, L, tokens
        self.depth = depth
        self.model, self.f, self.n_heads = model, ffn or 4 * h, n_heads
        self.n_layer = h * h if model == "mlp" else block_numel(h, self.f)
        assert all(x.numel >= self.n_layer for x in rc.infos), "registered layers too small for the model"
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.comm = comm_stream or torch.cuda.Stream(device=dev)
        self.comp = compute_stream or torch.cuda.current_stream(dev)
        npad = max(x.numel_pad for x in rc.infos)
        self.ring = GatherRing(max(n_bufs, depth + 2), npad, torch.bfloat16, dev)
        self.adam = H.make_adam(lr=lr)
        # gradient slots: bf16 (f4) or fp32 (qgZ quantizes fp32 gradients), zeroed once
        # (padding must stay zero)
        self.grad_dtype = grad_dtype
        self.gslots = []
        for i in range(L):
            ptr, n = H.hpz_buffer(self.ctx, i, "grad_slot")
            v = device_view(ptr, n, grad_dtype)
            v.zero_()
            self.gslots.append(v)
        self.k = 0          # gather sequence number (ring position)

    # -- Alg. 1 PrefetchAllGather -----------------------------------------------------
    def _gather(self, i: int, phase: str) -> int:
        b = self.ring.slot(self.k)
        self.k += 1
        if self.ring.free[b] is not None:
            self.comm.wait_event(self.ring.free[b])          # WAR: the buffer's last reader is done
        fn = H.hpz_fwd_gather if phase == "fwd" else H.hpz_bwd_gather
        fn(self.ctx, i, self.ring.bufs[b].data_ptr(), self.comm)
        self.ring.ready[b].record(self.comm)
        return b

    def _weights(self, b: int) -> torch.Tensor:
        self.comp.wait_event(self.ring.ready[b])              # "Ensure AllGather(L_i) finished"
        return self.ring.bufs[b][: self.h * self.h].view(self.h, self.h)

    def _release(self, b: int):
        ev = torch.cuda.Event()
        ev.record(self.comp)
        self.ring.free[b] = ev                                  # repartition(P)

    def step(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        if self.model == "transformer":
            return self._step_transformer(x, y)
        L = self.L
        with torch.cuda.stream(self.comp):
            # forward
            pending = {}
            for i in range(min(self.depth, L)):
                pending[i] = self._gather(i, "fwd")
            acts, pre = [x], []
            h = x
            for i in range(L):
                if i not in pending:
                    pending[i] = self._gather(i, "fwd")
                if i + self.depth < L and i + self.depth not in pending:
                    pending[i + self.depth] = self._gather(i + self.depth, "fwd")   # prefetch
                b = pending.pop(i)
                W = self._weights(b)
                z = h @ W.t()
                self._release(b)
                pre.append(z)
                h = torch.relu(z) if i < L - 1 else z
                acts.append(h)
            diff = h.float() - y.float()
            loss = (diff * diff).mean()
            dh = (2.0 / diff.numel() * diff).to(torch.bfloat16)
            # backward
            pending = {}
            for i in range(L - 1, max(L - 1 - self.depth, -1), -1):
                pending[i] = self._gather(i, "bwd")
            for i in reversed(range(L)):
                if i not in pending:
                    pending[i] = self._gather(i, "bwd")
                j = i - self.depth
                if j >= 0 and j not in pending:
                    pending[j] = self._gather(j, "bwd")                         # prefetch
                b = pending.pop(i)
                W = self._weights(b)
                dz = dh if i == L - 1 else dh * (pre[i] > 0).to(dh.dtype)
                slot = H.hpz_grad_buffer(self.ctx, i, self.comp)               # E6 on the compute stream
                dW = self.gslots[i][: self.h * self.h].view(self.h, self.h)
                if self.grad_dtype == "bf16":
                    torch.matmul(dz.t(), acts[i], out=dW)                       # L_i.backward() -> grad slot
                else:
                    dW.copy_(dz.t() @ acts[i])
                dh = dz @ W                                                      # uses the bwd-gathered W_i
                self._release(b)
                assert slot == self.gslots[i].data_ptr()
                g_ev = torch.cuda.Event()
                g_ev.record(self.comp)
                self.comm.wait_event(g_ev)
                H.hpz_reduce_scatter_adam(self.ctx, i, self.adam, self.comm)   # RS + optimizer.step()
        return loss

    def _step_transformer(self, x: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        """x, y: (B, S, h) bf16.  Same prefetch schedule as the MLP; per block the forward
        runs without autograd (input kept), the backward recomputes it under autograd from
        the backward-gathered parameters."""
        L, n = self.L, self.n_layer
        fwd = lambda flat, t: block_forward(flat, t, self.h, self.f, self.n_heads)   # noqa: E731
        with torch.cuda.stream(self.comp):
            pending = {}
            for i in range(min(self.depth, L)):
                pending[i] = self._gather(i, "fwd")
            acts = []
            hcur = x
            with torch.no_grad():
                for i in range(L):
                    if i not in pending:
                        pending[i] = self._gather(i, "fwd")
                    if i + self.depth < L and i + self.depth not in pending:
                        pending[i + self.depth] = self._gather(i + self.depth, "fwd")
                    b = pending.pop(i)
                    self.comp.wait_event(self.ring.ready[b])
                    acts.append(hcur)
                    hcur = fwd(self.ring.bufs[b][:n], hcur)
                    self._release(b)
            diff = hcur.float() - y.float()
            loss = (diff * diff).mean()
            dh = (2.0 / diff.numel() * diff).to(torch.bfloat16)
            pending = {}
            for i in range(L - 1, max(L - 1 - self.depth, -1), -1):
                pending[i] = self._gather(i, "bwd")
            for i in reversed(range(L)):
                if i not in pending:
                    pending[i] = self._gather(i, "bwd")
                j = i - self.depth
                if j >= 0 and j not in pending:
                    pending[j] = self._gather(j, "bwd")
                b = pending.pop(i)
                self.comp.wait_event(self.ring.ready[b])
                flat = self.ring.bufs[b][:n].detach().requires_grad_(True)   # backward-gathered W_i
                xin = acts[i].detach().requires_grad_(True)
                out = fwd(flat, xin)                                         # recompute (checkpoint)
                gflat, dh = torch.autograd.grad(out, (flat, xin), dh)
                slot = H.hpz_grad_buffer(self.ctx, i, self.comp)            # E6 on the compute stream
                assert slot == self.gslots[i].data_ptr()
                self.gslots[i][:n].copy_(gflat)                              # L_i.backward() -> grad slot
                self._release(b)
                g_ev = torch.cuda.Event()
                g_ev.record(self.comp)
                self.comm.wait_event(g_ev)
                H.hpz_reduce_scatter_adam(self.ctx, i, self.adam, self.comm)   # RS + optimizer.step()
        return loss
