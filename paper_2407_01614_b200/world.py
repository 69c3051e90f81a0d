"""Process/GPU plumbing around libhpz: one context per rank.

Two ways to build a world, both ending in the same C-ABI calls:

* ``DistWorld`` — the production path: one process per GPU (torchrun), every rank
  allocates its arena in libhpz, exchanges CUDA IPC handles through
  ``torch.distributed`` (``all_gather_object``; control plane only) and opens its
  peers' arenas as NVLink mappings.  No data ever moves through torch.distributed.
* ``EmulatedWorld`` — P ranks as P contexts in ONE process on ONE GPU, arenas bound
  to each other directly.  Every rank's operation is issued on one stream in SPMD
  round-robin order, so no kernel ever waits for a kernel that is not already ahead
  of it in the stream (B200_PROFILING.md: never run mutually-waiting kernels as
  separate launches on one GPU).  Used by the single-GPU parity tests.

``run_step`` drives one training step of Algorithm 1 for the
ranks a process owns.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import torch

from . import hpz as H

DTYPES = {"bf16": (H.HPZ_BF16, torch.bfloat16, 2), "f32": (H.HPZ_F32, torch.float32, 4)}


@dataclass
class RankCtx:
    ctx: object
    rank: int
    world: int
    node_size: int
    numels: list[int]
    infos: list = field(default_factory=list)

    def layer(self, i):
        return self.infos[i]


def virtual_nodes(world: int, node_size: int) -> list[list[int]]:
    """Consecutive ranks form a virtual node (readings R3/R4): 2x4 = [[0..3], [4..7]]."""
    if world < 1 or node_size < 1 or world % node_size:
        raise ValueError(f"node_size {node_size} must divide world {world}")
    return [list(range(n * node_size, (n + 1) * node_size)) for n in range(world // node_size)]


def exchange_handles(handle: bytes, group=None) -> list[bytes]:
    """All ranks' CUDA IPC handles in rank order (control plane only; works on gloo or nccl)."""
    import torch.distributed as dist
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, handle, group=group)
    if any(not isinstance(h, (bytes, bytearray)) or len(h) != H.IPC_HANDLE_BYTES for h in handles):
        raise RuntimeError("malformed IPC handle from a peer")
    return [bytes(h) for h in handles]


def _reduce_device(device):
    """Where a host-scalar reduction runs: the given device on NCCL, the host on gloo."""
    import torch.distributed as dist
    return "cpu" if dist.get_backend() == "gloo" else device


def max_over_ranks(values: list[float], device=None) -> list[float]:
    """Element-wise max over all ranks (timing rule: max over ranks); identity without a PG."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=_reduce_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.tolist()


def sum_over_ranks(values: list[float], device=None) -> list[float]:
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(values)
    t = torch.tensor(values, dtype=torch.float64, device=_reduce_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t.tolist()


def _register(ctx, numels, dtype, align, n_grad_slots, qgz=False, grad_dtype="f32", qwz=False, alias_secondary=True):
    if not alias_secondary:
        H.hpz_set_option(ctx, "alias_secondary", 0)   # keep a separate secondary at P' == P
    if qgz:
        H.hpz_set_option(ctx, "qgz", 4)        # sizes the arena: must precede register
    if qwz:
        H.hpz_set_option(ctx, "qwz", 8)
    if grad_dtype != "f32":
        H.hpz_set_option(ctx, "grad_dtype", DTYPES[grad_dtype][0])
    code = DTYPES[dtype][0]
    nbytes = H.hpz_register_flat_params(ctx, numels, code, align, n_grad_slots)
    return nbytes


class EmulatedWorld:
    """P ranks on one GPU in one process (test harness for the multi-rank protocol)."""

    def __init__(self, numels, world, node_size, dtype="bf16", align=256, n_grad_slots=None,
                 device=0, timeout_s=20.0, qgz=False, grad_dtype="f32", qwz=False, alias_secondary=True):
        self.world, self.node_size, self.dtype = world, node_size, dtype
        self.numels = list(numels)
        self.ranks: list[RankCtx] = []
        for r in range(world):
            ctx = H.hpz_init(world, node_size, r, device)
            _register(ctx, self.numels, dtype, align, n_grad_slots, qgz, grad_dtype, qwz, alias_secondary)
            H.hpz_arena_alloc(ctx)
            H.hpz_set_timeout(ctx, timeout_s)
            self.ranks.append(RankCtx(ctx, r, world, node_size, self.numels))
        ptrs = [H.hpz_arena_ptr(rc.ctx, rc.rank) for rc in self.ranks]
        for rc in self.ranks:
            H.hpz_bind(rc.ctx, ptrs)
            rc.infos = [H.hpz_layer_info(rc.ctx, i) for i in range(len(self.numels))]
        torch.cuda.synchronize()

    def close(self):
        for rc in self.ranks:
            H.hpz_finalize(rc.ctx)
        self.ranks = []


class DistWorld:
    """This process's single rank of a torch.distributed world (one GPU per process)."""

    def __init__(self, numels, node_size, dtype="bf16", align=256, n_grad_slots=None, device=None,
                 group=None, timeout_s=20.0, qgz=False, grad_dtype="f32", qwz=False, alias_secondary=True):
        import torch.distributed as dist
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.node_size = node_size
        self.dtype = dtype
        self.numels = list(numels)
        dev = torch.cuda.current_device() if device is None else device
        ctx = H.hpz_init(self.world, node_size, self.rank, dev)
        self.arena_bytes = _register(ctx, self.numels, dtype, align, n_grad_slots, qgz, grad_dtype, qwz,
                                     alias_secondary)
        handle = H.hpz_arena_alloc(ctx)
        H.hpz_set_timeout(ctx, timeout_s)
        virtual_nodes(self.world, node_size)         # validates the topology early
        H.hpz_arena_open(ctx, exchange_handles(handle, group))
        torch.cuda.synchronize()
        dist.barrier(group=group)          # every arena's flags are zero before any release
        rc = RankCtx(ctx, self.rank, self.world, node_size, self.numels)
        rc.infos = [H.hpz_layer_info(ctx, i) for i in range(len(self.numels))]
        self.ranks = [rc]

    def close(self):
        for rc in self.ranks:
            H.hpz_finalize(rc.ctx)
        self.ranks = []


def full_buffers(world_obj, n_bufs: int = 1, device=None):
    """Caller-owned full-parameter buffers (N̂_max elements of the param dtype) per rank."""
    tdt = DTYPES[world_obj.dtype][1]
    nmax = max(rc.infos[i].numel_pad for rc in world_obj.ranks for i in range(len(rc.numels)))
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    return [[torch.empty(nmax, dtype=tdt, device=dev) for _ in range(n_bufs)] for _ in world_obj.ranks]


def run_step(ranks: list[RankCtx], fwd_out, bwd_out, adam, stream=None, grad_fn=None,
             emulated: bool = False, layer_hook=None, fused: bool = False):
    """One step of Algorithm 1 for the given ranks (all P in emulation, or this process's one).

    fused=True replaces each layer's reduce-scatter and the final optimizer step by the
    fused per-layer RS+Adam kernel (same bits).
    fwd_out[r](i) / bwd_out[r](i) return the device pointer of the caller-owned full buffer
    for rank r, layer i.  grad_fn(rank_ctx, i) fills the rank's gradient slot (or None:
    gradients already resident).  In emulation every phase is issued for all ranks before
    the next phase, in the SPMD order of the real world."""
    L = len(ranks[0].numels)
    for i in range(L):                                      # forward, i = 1..N
        for rc in ranks:
            H.hpz_fwd_gather(rc.ctx, i, fwd_out[rc.rank](i), stream)
        if layer_hook:
            layer_hook("fwd", i)
    for i in reversed(range(L)):                            # backward, i = N..1
        for rc in ranks:
            H.hpz_bwd_gather(rc.ctx, i, bwd_out[rc.rank](i), stream)
        if layer_hook:
            layer_hook("bwd", i)
        if grad_fn is not None:
            for rc in ranks:
                grad_fn(rc, i)
        if emulated:
            for rc in ranks:
                H.hpz_grads_ready(rc.ctx, i, stream)
        for rc in ranks:
            if fused:                                       # RS + this layer's Adam, one kernel
                H.hpz_reduce_scatter_adam(rc.ctx, i, adam, stream)
            else:
                H.hpz_reduce_scatter(rc.ctx, i, stream)
        if layer_hook:
            layer_hook("rs", i)
    if not fused:
        for rc in ranks:                                    # optimizer.step()
            H.hpz_step(rc.ctx, -1, adam, stream)


class _CAI:
    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def device_view(ptr: int, n: int, dtype: str) -> torch.Tensor:
    """Zero-copy torch view of n elements at a device address in an arena.
    dtype: 'f32' -> float32, 'bf16' -> int16 bits viewed as bfloat16, 'u16'/'u32' bit views."""
    ts = {"f32": "<f4", "bf16": "<i2", "u16": "<i2", "u32": "<i4"}[dtype]
    t = torch.as_tensor(_CAI(ptr, n, ts), device="cuda")
    return t.view(torch.bfloat16) if dtype == "bf16" else t


def buffer_view(rc: RankCtx, layer: int, kind: str, dtype: str) -> torch.Tensor:
    ptr, n = H.hpz_buffer(rc.ctx, layer, kind)
    if kind in ("primary", "secondary") and dtype == "bf16":
        return device_view(ptr, n, "u16")
    if kind in ("primary", "secondary"):
        return device_view(ptr, n, "u32")
    return device_view(ptr, n, "f32")


def save_checkpoint(rc: RankCtx, adam_steps_done: int) -> dict:
    """This rank's optimizer state (SURVEY §5 checkpoint/resume): fp32 master, Adam m and v
    shards of every layer (CPU tensors) + the Adam step count."""
    torch.cuda.synchronize()
    state = {"rank": rc.rank, "world": rc.world, "node_size": rc.node_size, "numels": list(rc.numels),
             "shards": [int(x.shard) for x in rc.infos], "numel_pad": [int(x.numel_pad) for x in rc.infos],
             "adam_steps_done": int(adam_steps_done), "layers": []}
    for i in range(len(rc.numels)):
        state["layers"].append({k: buffer_view(rc, i, k, "f32").cpu().clone() for k in ("master", "m", "v")})
    return state


def load_checkpoint(rc: RankCtx, state: dict, stream=None):
    """Restore a save_checkpoint() state into a fresh context of the same layout/rank."""
    if state["rank"] != rc.rank or state["world"] != rc.world or list(state["numels"]) != list(rc.numels):
        raise ValueError("checkpoint was written for a different rank / world / model")
    # the shard geometry (padding: align_elems) must match too — hpz_load_state copies
    # `shard` fp32 elements per buffer from the given pointers
    if list(state.get("shards", [])) != [int(x.shard) for x in rc.infos] or \
            list(state.get("numel_pad", [])) != [int(x.numel_pad) for x in rc.infos]:
        raise ValueError("checkpoint was written with a different shard layout (align_elems)")
    keep = []
    for i, L in enumerate(state["layers"]):
        ts = [L[k].contiguous().cuda() for k in ("master", "m", "v")]
        for k, tk in zip(("master", "m", "v"), ts):
            if tk.dtype != torch.float32 or tk.numel() != rc.infos[i].shard:
                raise ValueError(f"checkpoint layer {i} {k}: expected {rc.infos[i].shard} fp32 elements")
        keep += ts
        H.hpz_load_state(rc.ctx, i, ts[0].data_ptr(), ts[1].data_ptr(), ts[2].data_ptr(),
                         state["adam_steps_done"], stream)
    torch.cuda.synchronize()
