"""Helpers shared by the -m gpu tests (test infrastructure: may use the oracle)."""
from __future__ import annotations

import numpy as np
import torch

from oracle import hpz_oracle as O
from synth import inputs as S


def gpu_ok() -> bool:
    return torch.cuda.is_available()


def bits_np(t: torch.Tensor, dtype: str) -> np.ndarray:
    a = t.detach().cpu()
    if dtype == "bf16":
        return a.view(torch.int16).numpy().view(np.uint16)
    return a.view(torch.int32).numpy().view(np.uint32) if a.dtype == torch.float32 else a.numpy().view(np.uint32)


def oracle_prim_bits(x: np.ndarray, dtype: str) -> np.ndarray:
    return O.param_bits(x, dtype)


def bits_equal(got: np.ndarray, want: np.ndarray, dtype: str) -> bool:
    """Bitwise equality with NaNs compared by class, never by payload (reading R10: the GPU's
    cvt / IEEE ops produce the canonical NaN, the oracle may keep an input's payload)."""
    got, want = np.asarray(got), np.asarray(want)
    if got.shape != want.shape:
        return False
    same = got == want
    if same.all():
        return True
    return bool((same | (O.is_nan_bits(got, dtype) & O.is_nan_bits(want, dtype))).all())


class ParityRun:
    """Drive an EmulatedWorld and an HpzOracle side by side on the same seeded inputs."""

    def __init__(self, numels, world, node_size, dtype="bf16", align=256, order="fixed",
                 verify="exact", grad_kind="uniform", n_grad_slots=None, stock_schedule="program",
                 fused=False, store_grad_shard=True, copy_engine="tma", qgz=False, grad_dtype="f32",
                 qwz=False, load_initial=True, init_params=None, grad_override=None):
        from paper_2407_01614_b200 import hpz as H
        from paper_2407_01614_b200.world import EmulatedWorld
        self.H = H
        self.numels, self.P, self.Pp, self.dtype = list(numels), world, node_size, dtype
        self.grad_kind = grad_kind
        self.fused, self.store_grad_shard = fused, store_grad_shard
        self.qgz, self.grad_dtype, self.qwz = qgz, grad_dtype, qwz
        self.w = EmulatedWorld(numels, world, node_size, dtype=dtype, align=align, n_grad_slots=n_grad_slots,
                               timeout_s=10.0, qgz=qgz, grad_dtype=grad_dtype, qwz=qwz)
        self.o = O.HpzOracle(self.numels, world, node_size, align=align, param_dtype=dtype,
                             order="fixed" if order == "paper" else order,
                             stock_schedule=stock_schedule, grad_kind=grad_kind, qgz=qgz, grad_dtype=grad_dtype,
                             qwz=qwz, init_params=init_params, grad_override=grad_override)
        self.init_params, self.grad_override = init_params, grad_override
        self.stream = torch.cuda.current_stream()
        for rc in self.w.ranks:
            H.hpz_set_order(rc.ctx, order)
            H.hpz_set_verify(rc.ctx, verify)
            H.hpz_set_option(rc.ctx, "store_grad_shard", int(store_grad_shard))
            H.hpz_set_option(rc.ctx, "copy_engine", H.COPY[copy_engine])
        tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
        L = len(self.numels)
        self.fwd = [[torch.zeros(rc.infos[i].numel_pad, dtype=tdt, device="cuda") for i in range(L)]
                    for rc in self.w.ranks]
        self.bwd = [[torch.zeros(rc.infos[i].numel_pad, dtype=tdt, device="cuda") for i in range(L)] for rc in self.w.ranks]
        for i, n in enumerate(self.numels if load_initial else []):
            w0 = torch.from_numpy(np.ascontiguousarray(init_params[i][:n], dtype=np.float32) if init_params is not None
                                  else S.layer_params(i, n)).cuda()
            for rc in self.w.ranks:
                H.hpz_load_master(rc.ctx, i, w0.data_ptr(), self.stream)
        self.adam = H.make_adam()
        self.t = 0

    def grads(self, i, t, r) -> np.ndarray:
        """Rank r's full-length (padded) fp32 gradient of layer i at step t, as uploaded."""
        lay = self.o.layouts[i]
        if self.grad_override is not None:
            return O.pad_full(np.asarray(self.grad_override(t, r, i), dtype=np.float32)[: lay.numel], lay)
        return S.layer_grads(i, t, r, lay.numel, lay.numel_pad, kind=self.grad_kind)

    def grad_fn(self, rc, i):
        lay = self.o.layouts[i]
        g = torch.from_numpy(np.ascontiguousarray(self.grads(i, self.t, rc.rank)[: lay.numel])).cuda()
        if self.grad_dtype == "bf16":
            g = g.to(torch.bfloat16)          # RNE, the same rounding as the oracle's bf16_rne
        self.H.hpz_grad_upload(rc.ctx, i, g.data_ptr(), lay.numel, self.stream)
        self._keep.append(g)

    def step(self, run_oracle=True):
        from paper_2407_01614_b200.world import run_step
        self._keep = []
        run_step(self.w.ranks, [lambda i, r=r: self.fwd[r][i].data_ptr() for r in range(self.P)],
                 [lambda i, r=r: self.bwd[r][i].data_ptr() for r in range(self.P)], self.adam,
                 stream=self.stream, grad_fn=self.grad_fn, emulated=True, fused=self.fused)
        torch.cuda.synchronize()
        rec = self.o.step() if run_oracle else None
        self.t += 1
        return rec

    def counters(self, reset=True):
        tot = {}
        for rc in self.w.ranks:
            c = self.H.hpz_counters(rc.ctx, reset=reset)
            for k, v in c.items():
                tot[k] = tot.get(k, 0) + v
        return tot

    def close(self):
        self.w.close()
