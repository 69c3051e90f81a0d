"""CPU oracle of the ZeRO++ hpZ data-parallel hot path (arXiv 2407.01614).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product (``paper_2407_01614_b200``) never imports it and shares no
code with it: not the layout math, not the reduction order, not the optimizer,
not the bf16 rounding.  The only thing both sides use is the seeded input
generator in ``synth/inputs.py``, which holds none of the method's arithmetic.

Plain, slow and obviously correct: numpy arrays, one rank at a time, Algorithm 1
step by step.  All P ranks are simulated in one process.  Citations are
``PAPER.md:<line>`` (the paper's LaTeX source) and ``SPEC.md:<line>``; readings
where the paper is silent are numbered R1..R25 as in DESIGN.md §3.

Precision: the paper never states one (R9).  Following BASELINE.json's
north_star, parameters are gathered in bf16 (toy config: fp32), gradients,
reduction and Adam run in fp32.  Because the north_star asks for bit-exact
gathers and a bit-exact fp32 reduce-scatter "in the same fixed reduction
order", the oracle evaluates those in fp32 in the fixed order (R7); fp64 is
used where the method has no fixed precision (toy-MLP forward/backward, the
float64 reference sums in the pins).

Pins (what ties this file to something other than itself) live in
``tests/test_oracle_*.py``; every function below names its pins.  Parity status:
every function is pinned; none is "parity unpinned".
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32

# ----------------------------------------------------------------------------
# a1. Layout and shard indexing  (Eq. (1); Alg. 1 Require,
#     PAPER.md:79-82; SPEC.md:276-297 partition examples; padding reading R2)
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class LayerLayout:
    """Shard geometry of one flat layer buffer.

    numel      N_i, the element count of the layer (R1: the "N" of Eq. (1))
    numel_pad  N̂_i = ceil(N_i / (P*A)) * P * A      (R2: one padding so that the
               secondary partition nests the primary one)
    shard      s_i  = N̂_i / P                       (primary, ZeRO-3)
    sec_shard  s'_i = N̂_i / P'                      (Eq. (1): |L_i,second| = N / secondaryWorldSize)
    Pins: tests/test_oracle_layout.py (SPEC examples with A=1, brute-force round
    trip, Eq. (1) size bound, BASELINE C2 numbers).
    """
    numel: int
    world: int
    node_size: int
    align: int

    @property
    def numel_pad(self) -> int:
        q = self.world * self.align
        return -(-self.numel // q) * q

    @property
    def shard(self) -> int:
        return self.numel_pad // self.world

    @property
    def sec_shard(self) -> int:
        return self.numel_pad // self.node_size


def check_topology(world: int, node_size: int) -> None:
    """P' must divide P and both be positive."""
    if world < 1 or node_size < 1 or world % node_size != 0:
        raise ValueError(f"invalid topology world={world} node_size={node_size}")


def node_of(rank: int, node_size: int) -> int:
    """n(r) = floor(r / P'): consecutive ranks form a (virtual) node (R4)."""
    return rank // node_size


def local_of(rank: int, node_size: int) -> int:
    """l(r) = r mod P': the rank's slice index inside its node (R3)."""
    return rank % node_size


def node_group(rank: int, node_size: int) -> list[int]:
    """The secondary group of ``rank``: the P' ranks of its node."""
    n = node_of(rank, node_size)
    return list(range(n * node_size, (n + 1) * node_size))


def pad_full(w: np.ndarray, lay: LayerLayout) -> np.ndarray:
    """Zero-pad a length-N_i buffer to N̂_i ("zero-padded")."""
    out = np.zeros(lay.numel_pad, dtype=w.dtype)
    out[: lay.numel] = w
    return out


def partition_primary(full_padded: np.ndarray, lay: LayerLayout, rank: int) -> np.ndarray:
    """Rank r's contiguous primary shard [r*s, (r+1)*s) (ZeRO-3)."""
    s = lay.shard
    return full_padded[rank * s:(rank + 1) * s].copy()


# ----------------------------------------------------------------------------
# a2 / a4. Gathers and the secondary copy (Alg. 1 PAPER.md:87, 94, 101-105, 110;
#          Eq. (1) text PAPER.md:128)
# ----------------------------------------------------------------------------


def all_gather(shards: list[np.ndarray]) -> np.ndarray:
    """AllGather = concatenation of the group's shards in rank order.
    Pins: concatenation example, round trip, gather of constant shards."""
    return np.concatenate(shards)


def secondary_copy(full: np.ndarray, lay: LayerLayout, rank: int) -> np.ndarray:
    """Alg. 1: L_i,second <- empty(|L_i|/P'); copy the local rank's
    slice of the full parameter tensor.  Slice l(r) of size s'.
    Pins: Eq. (1) examples, secondary == concat of primaries."""
    sp = lay.sec_shard
    l = local_of(rank, lay.node_size)
    return full[l * sp:(l + 1) * sp].copy()


def fwd_gather(prims: list[np.ndarray]) -> np.ndarray:
    """Forward: AllGather(L_i, P) over the primary shards."""
    return all_gather(prims)


def bwd_gather(secs: list[np.ndarray], lay: LayerLayout, rank: int) -> np.ndarray:
    """Backward: AllGather(L_i, P') over the secondary shards of rank's node."""
    return all_gather([secs[q] for q in node_group(rank, lay.node_size)])


# ----------------------------------------------------------------------------
# a5. Gradient reduce-scatter (Alg. 1 PAPER.md:115 "ReduceScatter(∇L_i, P)")
#     Mean (R6); fixed pairwise-by-rank association (R7).
# ----------------------------------------------------------------------------


def pairwise_rank_sum(vals: list[np.ndarray]) -> np.ndarray:
    """Fixed association (R7): sum adjacent rank pairs level by level,
    [(G0+G1), (G2+G3), ...], an odd last operand carried to the next level,
    until one value is left.  For P=8: ((G0+G1)+(G2+G3))+((G4+G5)+(G6+G7)).
    Every addition is one fp32 IEEE round-to-nearest add.
    Pins: dyadic-grid exact closed form, float64 error bound, DP consistency."""
    level = [np.asarray(v, dtype=F32) for v in vals]
    while len(level) > 1:
        nxt = [(level[2 * k] + level[2 * k + 1]).astype(F32) for k in range(len(level) // 2)]
        if len(level) % 2:
            nxt.append(level[-1])
        level = nxt
    return level[0]


def reduce_scatter(grads: list[np.ndarray], lay: LayerLayout, rank: int) -> np.ndarray:
    """Rank r's fp32 gradient shard g_r[e] = (Σ_j G_j[r*s+e]) * (1/P).
    The sum uses the fixed association of ``pairwise_rank_sum``; 1/P is exact
    for power-of-two P.  Pins: SPEC example P=2 [1,1],[3,3] -> [2],[2]; P=1 identity."""
    s = lay.shard
    parts = [np.asarray(g[rank * s:(rank + 1) * s], dtype=F32) for g in grads]
    total = pairwise_rank_sum(parts)
    return (total * F32(1.0 / lay.world)).astype(F32)


# ----------------------------------------------------------------------------
# bf16 round-to-nearest-even (R10)
# ----------------------------------------------------------------------------


def bf16_rne(x: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits (uint16), round to nearest, ties to even; overflow -> inf;
    NaN -> a quiet NaN (payload unspecified: compare NaNs by class, R10).
    Pins: tie cases 0x3f808000->0x3f80, 0x3f818000->0x3f82, 0x7f7fffff->0x7f80,
    and agreement with torch's CPU bfloat16 cast on random finite values."""
    u = np.asarray(x, dtype=F32).view(np.uint32).astype(np.uint64)
    exp_all_ones = (u & 0x7F800000) == 0x7F800000
    is_nan = exp_all_ones & ((u & 0x007FFFFF) != 0)
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) & 0xFFFF
    r = np.where(is_nan, (u >> 16) | 0x0040, r)
    return r.astype(np.uint16)


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << 16).view(F32)


def is_nan_bits(bits: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        b = np.asarray(bits, dtype=np.uint16)
        return ((b & 0x7F80) == 0x7F80) & ((b & 0x007F) != 0)
    b = np.asarray(bits, dtype=np.uint32)
    return ((b & 0x7F800000) == 0x7F800000) & ((b & 0x007FFFFF) != 0)


# ----------------------------------------------------------------------------
# a6. Partitioned Adam + primary refresh (Alg. 1 PAPER.md:117 "optimizer.step()";
#     sharded optimizer states PAPER.md:64; Adam per north_star, R8)
# ----------------------------------------------------------------------------


@dataclass(frozen=True)
class AdamHyper:
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    weight_decay: float = 0.0


@dataclass(frozen=True)
class AdamScalars:
    """Per-step fp32 scalars, computed in float64 and rounded once (R8, R24)."""
    beta1: np.float32
    beta2: np.float32
    omb1: np.float32
    omb2: np.float32
    step_size: np.float32   # lr / (1 - beta1^t)
    bc2_sqrt: np.float32    # sqrt(1 - beta2^t)
    eps: np.float32
    lr_wd: np.float32       # lr * weight_decay (decoupled, AdamW form)


def adam_scalars(h: AdamHyper, t_adam: int) -> AdamScalars:
    """t_adam is the 1-based Adam step count (R24)."""
    if t_adam < 1:
        raise ValueError("Adam step count is 1-based")
    bc1 = 1.0 - h.beta1 ** t_adam
    bc2 = 1.0 - h.beta2 ** t_adam
    return AdamScalars(F32(h.beta1), F32(h.beta2), F32(1.0 - h.beta1), F32(1.0 - h.beta2),
                       F32(h.lr / bc1), F32(math.sqrt(bc2)), F32(h.eps),
                       F32(h.lr * h.weight_decay))


def adam_update(w: np.ndarray, m: np.ndarray, v: np.ndarray, g: np.ndarray,
                sc: AdamScalars) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """One Adam step (Kingma & Ba, bias-corrected), elementwise, fp32, in exactly this
    order, each line a single IEEE operation per binary operator (no fused multiply-add):

        m = beta1*m + (1-beta1)*g
        v = beta2*v + ((1-beta2)*g)*g
        d = sqrt(v)/sqrt(1-beta2^t) + eps
        w = w - lr*wd*w                  (only if wd != 0; decoupled decay)
        w = w - (lr/(1-beta1^t)) * (m/d)

    Pins: t=1 closed form |Δw| = lr*|g|/(|g|+eps); lr=0 no-op; torch.optim.Adam in
    float64 within 1e-6 relative; partitioned == unpartitioned."""
    w = np.asarray(w, dtype=F32)
    g = np.asarray(g, dtype=F32)
    m = (sc.beta1 * np.asarray(m, dtype=F32) + sc.omb1 * g).astype(F32)
    v = (sc.beta2 * np.asarray(v, dtype=F32) + (sc.omb2 * g).astype(F32) * g).astype(F32)
    d = (np.sqrt(v) / sc.bc2_sqrt + sc.eps).astype(F32)
    if sc.lr_wd != 0:
        w = (w - sc.lr_wd * w).astype(F32)
    w = (w - sc.step_size * (m / d).astype(F32)).astype(F32)
    return w, m, v


def sgd_update(w: np.ndarray, g: np.ndarray, lr: float) -> np.ndarray:
    """Plain SGD w <- w - lr*g, used only in the brute-force pins."""
    return (np.asarray(w, dtype=F32) - F32(lr) * np.asarray(g, dtype=F32)).astype(F32)


def refresh_primary(master: np.ndarray, param_dtype: str) -> np.ndarray:
    """Primary = master rounded to the parameter dtype (bf16 RNE, R10; fp32 copy)."""
    if param_dtype == "bf16":
        return bf16_rne(master)
    return np.asarray(master, dtype=F32).copy()


def param_bits(x: np.ndarray, param_dtype: str) -> np.ndarray:
    """Bit pattern of a parameter buffer (uint16 for bf16 storage, uint32 for fp32)."""
    if param_dtype == "bf16":
        return np.asarray(x, dtype=np.uint16)
    return np.asarray(x, dtype=F32).view(np.uint32)


def param_values(x: np.ndarray, param_dtype: str) -> np.ndarray:
    if param_dtype == "bf16":
        return bf16_to_f32(x)
    return np.asarray(x, dtype=F32)


POISON_BF16 = np.uint16(0x7FC0)       # R16: "arbitrarily initialized" -> quiet NaN
POISON_F32 = np.uint32(0x7FC00000)


def poison_like(n: int, param_dtype: str) -> np.ndarray:
    """torch.empty analog (SPEC NanFill SPEC.md:48)."""
    if param_dtype == "bf16":
        return np.full(n, POISON_BF16, dtype=np.uint16)
    return np.full(n, POISON_F32, dtype=np.uint32).view(F32)


# ----------------------------------------------------------------------------
# C1 toy model: 2-layer MLP 512 -> 1024 -> 512, tanh, MSE vs a teacher
# Forward/backward in float64; grads handed to the reduce-scatter as fp32.
# Pins: central finite differences; loss decreases; DP consistency.
# ----------------------------------------------------------------------------

TOY_DIMS = (512, 1024, 512)


def toy_layer_numels(dims=TOY_DIMS) -> list[int]:
    """fc1: W1 (h x d) row-major then b1 (h); fc2: W2 (o x h) then b2 (o)."""
    d, h, o = dims
    return [h * d + h, o * h + o]


def toy_unflatten(flat: list[np.ndarray], dims=TOY_DIMS):
    d, h, o = dims
    f1, f2 = (np.asarray(x, dtype=np.float64) for x in flat)
    W1 = f1[: h * d].reshape(h, d)
    b1 = f1[h * d: h * d + h]
    W2 = f2[: o * h].reshape(o, h)
    b2 = f2[o * h: o * h + o]
    return W1, b1, W2, b2


def toy_loss_and_grads(flat_fwd: list[np.ndarray], flat_bwd: list[np.ndarray],
                       x: np.ndarray, y: np.ndarray, dims=TOY_DIMS):
    """Loss = mean((f(x) - y)^2) with f(x) = W2 tanh(W1 x + b1) + b2.

    ``flat_fwd`` are the forward-gathered layer buffers (Alg. 1),
    ``flat_bwd`` the backward-gathered ones: the backward pass
    multiplies by the weights it gathered, so a stale or garbage secondary
    reaches the gradients exactly as in the paper's failure.
    Returns (loss, [g_fc1, g_fc2]) with unpadded float64 gradients."""
    W1, b1, W2, b2 = toy_unflatten(flat_fwd, dims)
    W1b, _, W2b, _ = toy_unflatten(flat_bwd, dims)
    x = np.asarray(x, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    B = x.shape[0]
    z1 = x @ W1.T + b1
    a1 = np.tanh(z1)
    out = a1 @ W2.T + b2
    diff = out - y
    loss = float(np.mean(diff * diff))
    dout = 2.0 * diff / diff.size
    gW2 = dout.T @ a1
    gb2 = dout.sum(axis=0)
    da1 = dout @ W2b
    dz1 = da1 * (1.0 - a1 * a1)
    gW1 = dz1.T @ x
    gb1 = dz1.sum(axis=0)
    d, h, o = dims
    g1 = np.concatenate([gW1.reshape(-1), gb1])
    g2 = np.concatenate([gW2.reshape(-1), gb2])
    _ = B
    return loss, [g1, g2]


def toy_batch(step: int, rank: int, batch: int = 64, dims=TOY_DIMS, identical: bool = False):
    """Synthetic regression batch: inputs from the seeded generator, targets from a
    fixed random teacher of the same architecture."""
    from synth import inputs as S
    d, h, o = dims
    r = 0 if identical else rank
    x = S.uniform(S.stream_key(S.SEED_TOY_DATA, 1000, step, r), np.arange(batch * d), 1.0)
    x = x.reshape(batch, d).astype(np.float64)
    tw = [S.uniform(S.stream_key(S.SEED_TOY_DATA, 2000 + i, 0, 0), np.arange(n), 2.0 ** -4)
          for i, n in enumerate(toy_layer_numels(dims))]
    W1, b1, W2, b2 = toy_unflatten(tw, dims)
    y = np.tanh(x @ W1.T + b1) @ W2.T + b2
    return x, y


# ----------------------------------------------------------------------------
# The whole step: Algorithm 1 over all P ranks
# ----------------------------------------------------------------------------

ORDERS = ("fixed", "stock", "off")
STOCK_SCHEDULES = ("program", "adversarial_stale", "realloc", "half_written", "realistic")


def prefetch_enqueue_order(n_layers: int, depth: int) -> list[tuple]:
    """The operations Algorithm 1 enqueues in one step, in program order,
    with ZeRO-3 prefetch of `depth` modules (reading R12).  Modules execute in the order
    fwd L_1..L_N, bwd L_N..L_1.  For each module: "Ensure AllGather(L_i) finished" (an
    AllGather not prefetched earlier is enqueued now, on demand), PrefetchAllGather() (the
    AllGathers of the next `depth` modules not yet enqueued — forward ones over P, backward
    ones over P'), the module's compute, and — after a forward — "L_i,second <- empty; Copy to
    L_i,second (Async MemcpyD2D)".  Layers are 0-based.  Returns
    [("gather", "fwd"|"bwd", i) | ("copy", i), ...]."""
    modules = [("fwd", i) for i in range(n_layers)] + [("bwd", i) for i in reversed(range(n_layers))]
    seq, enq = [], set()
    for pos, m in enumerate(modules):
        if m not in enq:                                   # Ensure AllGather(L_i) finished
            enq.add(m)
            seq.append(("gather",) + m)
        for nxt in modules[pos + 1:pos + 1 + depth]:       # PrefetchAllGather()
            if nxt not in enq:
                enq.add(nxt)
                seq.append(("gather",) + nxt)
        if m[0] == "fwd":                                  # L_i.forward(); then the async copy
            seq.append(("copy", m[1]))
    return seq


def realistic_racing_layers(n_layers: int, depth: int) -> set[int]:
    """Layers whose backward AllGather(L_i, P') is ENQUEUED before their own secondary copy
    under Alg. 1 with prefetch depth `depth`: without the fix (stock ZeRO++) nothing orders
    the two, so the gather can read the secondary "still being partitioned" — the race of
    PAPER.md:130-132, at the forward->backward turnaround of Fig. 1.  Every
    other backward gather is enqueued after its copy (R13: in the realistic schedule those
    read the fresh copy).  Pins: tests/test_oracle_step.py (closed form: the last
    ceil(depth/2) layers, none without prefetch)."""
    seq = prefetch_enqueue_order(n_layers, depth)
    return {i for i in range(n_layers) if seq.index(("gather", "bwd", i)) < seq.index(("copy", i))}


@dataclass
class RankLayerState:
    prim: np.ndarray          # param dtype storage (uint16 bf16 bits or fp32), length s
    master: np.ndarray        # fp32, s
    m: np.ndarray             # fp32, s
    v: np.ndarray             # fp32, s
    sec: np.ndarray | None = None   # param dtype storage, length s' (persistent, R5)


@dataclass
class StepRecord:
    t: int
    W: list[np.ndarray]                 # W_t^i: full params gathered in forward (param storage)
    mismatches: list[int]               # per layer, summed over ranks
    nan_reads: list[int]
    loss: float | None = None


@dataclass
class HpzOracle:
    """All P ranks of the hpZ hot path, simulated literally.

    order: "fixed" (the paper's fix), "stock" (no wait, the bug,
    PAPER.md:130-132) or "off" (plain ZeRO-3: backward AllGather over P from
    the primaries, Table 1 "without hpZ").
    stock_schedule chooses how the unordered secondary copy interleaves with the
    backward gather (R5, R13): "program" (copy lands first), "adversarial_stale"
    (every backward read happens before this step's copy: persistent buffer holds
    the previous step's slice, poison at t=0), "realloc" (fresh torch.empty each
    step, read before the copy: poison), "half_written" (a seeded prefix refreshed),
    "realistic" (only the layers `realistic_racing_layers(N, prefetch_depth)` read before
    their copy — the previous step's slice, poison at t=0 — every other layer after it).
    """
    numels: list[int]
    world: int
    node_size: int
    align: int = 256
    param_dtype: str = "bf16"
    order: str = "fixed"
    stock_schedule: str = "program"
    hyper: AdamHyper = field(default_factory=AdamHyper)
    optimizer: str = "adam"
    grad_source: str = "synthetic"      # "synthetic" | "toy"
    grad_kind: str = "uniform"
    toy_identical_batches: bool = False
    half_seed: int = 1234
    prefetch_depth: int = 1              # "realistic" stock schedule (R12)
    # test inputs other than the seeded generator (no arithmetic of the method): the full
    # fp32 initial parameters of each layer, and a callable (t, rank, layer) -> the rank's
    # full-length fp32 gradient of the layer at step t (e.g. what a real backward wrote)
    init_params: list | None = None
    grad_override: object = None
    qgz: bool = False                    # f1: INT4 quantized gradient all-to-all (qgz_reduce_scatter)
    grad_dtype: str = "f32"              # f4: "bf16" = gradients stored/communicated as bf16 (RNE)
    qwz: bool = False                    # f2: INT8 blockwise weights in the forward AllGather

    def __post_init__(self):
        check_topology(self.world, self.node_size)
        if self.qwz and self.align % QWZ_BLOCK:
            raise ValueError("qwZ needs shards made of whole 256-element blocks (align % 256 == 0)")
        if self.order not in ORDERS or self.stock_schedule not in STOCK_SCHEDULES:
            raise ValueError("bad order/schedule")
        self.layouts = [LayerLayout(n, self.world, self.node_size, self.align) for n in self.numels]
        self.t = 0
        self.history: list[StepRecord] = []
        self.state: list[list[RankLayerState]] = []
        from synth import inputs as S
        for i, lay in enumerate(self.layouts):
            if self.grad_source == "toy":
                w0 = np.zeros(lay.numel_pad, dtype=F32)
                d, h, o = TOY_DIMS
                fan_in = d if i == 0 else h
                w0[: lay.numel] = S.uniform(S.stream_key(S.SEED_PARAMS, i, 0, 0),
                                            np.arange(lay.numel), 2.0 ** -int(math.log2(fan_in) / 2 + 1))
            elif self.init_params is not None:
                w0 = pad_full(np.asarray(self.init_params[i], dtype=F32)[: lay.numel], lay)
            else:
                w0 = S.layer_params(i, lay.numel, lay.numel_pad)
            ranks = []
            for r in range(self.world):
                master = partition_primary(w0, lay, r)
                ranks.append(RankLayerState(
                    prim=refresh_primary(master, self.param_dtype), master=master,
                    m=np.zeros(lay.shard, F32), v=np.zeros(lay.shard, F32),
                    sec=poison_like(lay.sec_shard, self.param_dtype)))
            self.state.append(ranks)

    # --- grads -------------------------------------------------------------
    def _grads(self, t: int, fwd_full: list[list[np.ndarray]], bwd_full: list[list[np.ndarray]]):
        """G[r][i]: full-length fp32 gradient of rank r for layer i (zero padding)."""
        from synth import inputs as S
        G = []
        losses = []
        for r in range(self.world):
            if self.grad_source == "toy":
                x, y = toy_batch(t, r, identical=self.toy_identical_batches)
                f = [param_values(fwd_full[i][r], self.param_dtype)[: lay.numel] for i, lay in enumerate(self.layouts)]
                b = [param_values(bwd_full[i][r], self.param_dtype)[: lay.numel] for i, lay in enumerate(self.layouts)]
                loss, gs = toy_loss_and_grads(f, b, x, y)
                losses.append(loss)
                G.append([pad_full(g.astype(F32), lay) for g, lay in zip(gs, self.layouts)])
            elif self.grad_override is not None:
                G.append([pad_full(np.asarray(self.grad_override(t, r, i), dtype=F32)[: lay.numel], lay)
                          for i, lay in enumerate(self.layouts)])
            else:
                G.append([S.layer_grads(i, t, r, lay.numel, lay.numel_pad, kind=self.grad_kind)
                          for i, lay in enumerate(self.layouts)])
            if self.grad_dtype == "bf16":     # f4: the slot holds bf16; widening to fp32 is exact
                G[-1] = [bf16_to_f32(bf16_rne(g)) for g in G[-1]]
        return G, (float(np.mean(losses)) if losses else None)

    # --- one training step (Alg. 1 While body) ---------------
    def step(self) -> StepRecord:
        t = self.t
        P = self.world
        L = len(self.layouts)
        rng = np.random.default_rng(self.half_seed + t)
        W_t, fwd_full, bwd_full = [], [], []
        mism = [0] * L
        nans = [0] * L
        # Forward pass, i = 1..N
        for i, lay in enumerate(self.layouts):
            prims = [self.state[i][r].prim for r in range(P)]
            if self.qwz:                                        # f2: quantize before AllGather
                prims = [qwz_gathered_shard(p_, self.param_dtype) for p_ in prims]
            F = [fwd_gather(prims) for _ in range(P)]          # AllGather(L_i, P), every rank
            for r in range(P):
                assert np.array_equal(param_bits(F[r], self.param_dtype), param_bits(F[0], self.param_dtype))
            W_t.append(F[0].copy())
            fwd_full.append(F)
            if self.order == "off":
                continue
            # L_i,second <- empty(|L_i|/P'); async copy
            racing = (realistic_racing_layers(L, self.prefetch_depth)
                      if self.stock_schedule == "realistic" else set())
            for r in range(P):
                st = self.state[i][r]
                fresh = secondary_copy(F[r], lay, r)
                if self.order == "fixed" or self.stock_schedule == "program" or \
                        (self.stock_schedule == "realistic" and i not in racing):
                    st.sec = fresh                      # the wait orders it
                elif self.stock_schedule in ("adversarial_stale", "realistic"):
                    st.pending = fresh                  # lands only after the backward read
                elif self.stock_schedule == "realloc":
                    st.sec = poison_like(lay.sec_shard, self.param_dtype)
                    st.pending = fresh
                elif self.stock_schedule == "half_written":
                    h = int(rng.integers(0, lay.sec_shard + 1))
                    part = st.sec.copy()
                    part[:h] = fresh[:h]
                    st.sec = part
                    st.pending = fresh
        # Backward gathers, i = N..1, then the pending copies land
        B_all = [None] * L
        for i in reversed(range(L)):
            lay = self.layouts[i]
            Bi = []
            for r in range(P):
                if self.order == "off":
                    B = fwd_gather([self.state[i][j].prim for j in range(P)])   # AllGather(L_i, P)
                else:
                    B = bwd_gather([self.state[i][q].sec for q in range(P)], lay, r)
                bits = param_bits(B, self.param_dtype)[: lay.numel]
                ref = param_bits(W_t[i], self.param_dtype)[: lay.numel]
                mism[i] += int(np.count_nonzero(bits != ref))
                nans[i] += int(np.count_nonzero(is_nan_bits(bits, self.param_dtype)))
                Bi.append(B)
            B_all[i] = Bi
        for i in range(L):
            for r in range(P):
                st = self.state[i][r]
                if hasattr(st, "pending"):
                    st.sec = st.pending
                    del st.pending
        bwd_full = B_all
        # L_i.backward() stand-in: gradients (synthetic, or the toy MLP on B_r)
        G, loss = self._grads(t, fwd_full, bwd_full)
        # ReduceScatter(∇L_i, P), then optimizer.step()
        for i, lay in enumerate(self.layouts):
            for r in range(P):
                rs = qgz_reduce_scatter if self.qgz else reduce_scatter
                g = rs([G[j][i] for j in range(P)], lay, r)
                st = self.state[i][r]
                if self.optimizer == "adam":
                    st.master, st.m, st.v = adam_update(st.master, st.m, st.v, g,
                                                        adam_scalars(self.hyper, t + 1))
                else:
                    st.master = sgd_update(st.master, g, self.hyper.lr)
                st.prim = refresh_primary(st.master, self.param_dtype)
        rec = StepRecord(t=t, W=W_t, mismatches=mism, nan_reads=nans, loss=loss)
        self.history.append(rec)
        self.t += 1
        return rec

    def run(self, steps: int) -> list[StepRecord]:
        return [self.step() for _ in range(steps)]

    # --- views -------------------------------------------------------------
    def full_master(self, i: int) -> np.ndarray:
        return np.concatenate([self.state[i][r].master for r in range(self.world)])

    def full_primary(self, i: int) -> np.ndarray:
        return np.concatenate([self.state[i][r].prim for r in range(self.world)])


# ----------------------------------------------------------------------------
# Unpartitioned reference (brute force, no shards): the pin for partitioning
# ----------------------------------------------------------------------------


def unpartitioned_train(numels: list[int], world: int, steps: int, hyper: AdamHyper,
                        param_dtype: str = "bf16", optimizer: str = "adam",
                        grad_source: str = "synthetic", init_full: list[np.ndarray] | None = None):
    """One process, full buffers, no sharding: per-rank grads (same generator), mean
    in the same fixed order, optimizer on the whole vector.  hpZ only changes the
    communication routing, not the math (Fig. 2 claim PAPER.md:207)."""
    from synth import inputs as S
    L = len(numels)
    if init_full is None:
        init_full = [S.layer_params(i, n) for i, n in enumerate(numels)]
    master = [np.asarray(w, dtype=F32).copy() for w in init_full]
    m = [np.zeros(n, F32) for n in numels]
    v = [np.zeros(n, F32) for n in numels]
    losses = []
    for t in range(steps):
        params = [param_values(refresh_primary(w, param_dtype), param_dtype) for w in master]
        if grad_source == "toy":
            per_rank = []
            ls = []
            for r in range(world):
                x, y = toy_batch(t, r)
                loss, gs = toy_loss_and_grads(params, params, x, y)
                ls.append(loss)
                per_rank.append([g.astype(F32) for g in gs])
            losses.append(float(np.mean(ls)))
        else:
            per_rank = [[S.layer_grads(i, t, r, numels[i]) for i in range(L)] for r in range(world)]
        for i in range(L):
            g = (pairwise_rank_sum([per_rank[r][i] for r in range(world)]) * F32(1.0 / world)).astype(F32)
            if optimizer == "adam":
                master[i], m[i], v[i] = adam_update(master[i], m[i], v[i], g, adam_scalars(hyper, t + 1))
            else:
                master[i] = sgd_update(master[i], g, hyper.lr)
    return master, m, v, losses


# ----------------------------------------------------------------------------
# Sampled evaluation at full size (parity at BASELINE sizes)
# ----------------------------------------------------------------------------


def sampled_trajectory(layer: int, numel: int, world: int, idx: np.ndarray, steps: int,
                       hyper: AdamHyper, param_dtype: str = "bf16", grad_scale: float | None = None,
                       fixed_grads: bool = False):
    """Master/m/v/primary at full-layer element indices ``idx`` after ``steps`` steps
    with synthetic gradients: every quantity of the path is elementwise in the
    element index once the layout is fixed, so a sample is computed one element
    at a time (same functions as the full simulation).  ``fixed_grads``: every step
    reuses the step-0 gradients (bench.py keeps its gradients resident)."""
    from synth import inputs as S
    gs = S.GRAD_SCALE if grad_scale is None else grad_scale
    idx = np.asarray(idx, dtype=np.int64)
    w = S.values_at(S.SEED_PARAMS, layer, 0, 0, idx, S.PARAM_SCALE, numel)
    m = np.zeros(idx.size, F32)
    v = np.zeros(idx.size, F32)
    for t in range(steps):
        tg = 0 if fixed_grads else t
        grads = [S.values_at(S.SEED_GRADS, layer, tg, r, idx, gs, numel) for r in range(world)]
        g = (pairwise_rank_sum(grads) * F32(1.0 / world)).astype(F32)
        w, m, v = adam_update(w, m, v, g, adam_scalars(hyper, t + 1))
    return w, m, v, refresh_primary(w, param_dtype)


# ----------------------------------------------------------------------------
# f1. qgZ: blockwise INT4 gradient quantization + all-to-all in place of the fp32
#     reduce-scatter ("quantizes gradients before ReduceScatter";
#     Alg. 1 comment PAPER.md:114 "Replaced with INT4 AllToAll if with qgZ").
#     The paper does not state the quantizer (it defers to ZeRO++); reading R26 takes
#     SPEC's asymmetric blockwise scheme: per block of 64 elements
#     min_b, scale_b = (max_b - min_b) / (2^bits - 1), code = round((v - min_b)/scale_b),
#     v̂ = min_b + code * scale_b.  fp32 throughout, one IEEE op per operator, round =
#     round-half-to-even, codes clamped to [0, 2^bits - 1].
# ----------------------------------------------------------------------------

QGZ_BITS = 4
QGZ_BLOCK = 64


def quantize_blockwise(v: np.ndarray, bits: int = QGZ_BITS, block: int = QGZ_BLOCK):
    """Returns (codes uint8 per element, mins fp32 per block, scales fp32 per block).
    A block containing NaN gets NaN min/scale (NaN must surface).
    Pins: SPEC examples (constant block -> scale 0, codes 0; [0, 1] at 8 bits -> codes
    [0, 255]); |v - v̂| <= scale/2 (+1 ulp slack) by brute force; monotone code map."""
    v = np.asarray(v, dtype=F32)
    if v.size % block:
        raise ValueError("length must be a multiple of the block")
    b = v.reshape(-1, block)
    nan_blk = np.isnan(b).any(axis=1)
    with np.errstate(invalid="ignore"):
        mins = np.where(nan_blk, np.float32(np.nan), np.nanmin(np.where(np.isnan(b), np.inf, b), axis=1)).astype(F32)
        maxs = np.where(nan_blk, np.float32(np.nan), np.nanmax(np.where(np.isnan(b), -np.inf, b), axis=1)).astype(F32)
        levels = F32((1 << bits) - 1)
        scales = ((maxs - mins).astype(F32) / levels).astype(F32)
        q = ((b - mins[:, None]).astype(F32) / scales[:, None]).astype(F32)
        codes = np.rint(q)
        codes = np.where(scales[:, None] > 0, codes, 0.0)
        codes = np.clip(np.nan_to_num(codes, nan=0.0), 0, (1 << bits) - 1).astype(np.uint8)
    return codes.reshape(-1), mins, scales


def dequantize_blockwise(codes: np.ndarray, mins: np.ndarray, scales: np.ndarray,
                         block: int = QGZ_BLOCK) -> np.ndarray:
    """v̂ = min_b + code * scale_b (fp32, multiply then add)."""
    c = np.asarray(codes, dtype=F32).reshape(-1, block)
    prod = (c * scales[:, None]).astype(F32)
    return (mins[:, None] + prod).astype(F32).reshape(-1)


def qgz_reduce_scatter(grads: list[np.ndarray], lay: LayerLayout, rank: int,
                       bits: int = QGZ_BITS, block: int = QGZ_BLOCK) -> np.ndarray:
    """Owner r's gradient shard under qgZ: every rank j quantizes its full gradient,
    the all-to-all delivers rank j's quantized slice [r*s, (r+1)*s) to owner r, which
    dequantizes each slice and reduces them in the fixed order of ``pairwise_rank_sum``,
    times 1/P.  Pins: within sum_j scale_j/2 / P of the fp32 reduce-scatter; exact when
    every block is constant."""
    s = lay.shard
    parts = []
    for g in grads:
        codes, mins, scales = quantize_blockwise(g, bits, block)
        b0, b1 = rank * s // block, (rank + 1) * s // block
        parts.append(dequantize_blockwise(codes[rank * s:(rank + 1) * s], mins[b0:b1], scales[b0:b1], block))
    total = pairwise_rank_sum(parts)
    return (total * F32(1.0 / lay.world)).astype(F32)


# ----------------------------------------------------------------------------
# f2. qwZ: blockwise INT8 weight quantization before the forward AllGather
#     ("the qwZ scheme quantizes weights before AllGather operations").
#     Reading R28 (the paper does not state the scheme): SPEC's asymmetric blockwise
#     quantizer with 8 bits and 256-element blocks (SPEC's qwZ default),
#     applied by the owner to its primary shard (the values as fp32); the forward gather
#     dequantizes (min + code*scale, fp32) and rounds to the parameter dtype (bf16 RNE).
#     The secondary is written from the forward-gathered values, so the backward gather
#     returns exactly what the forward gather returned.
# ----------------------------------------------------------------------------

QWZ_BITS = 8
QWZ_BLOCK = 256


def qwz_gathered_shard(prim: np.ndarray, param_dtype: str) -> np.ndarray:
    """What every rank receives for one owner's primary shard under qwZ (param storage).
    Pins: exact on constant blocks; within scale/2 (+ one bf16 rounding) of the primary."""
    vals = param_values(prim, param_dtype)
    codes, mins, scales = quantize_blockwise(vals, QWZ_BITS, QWZ_BLOCK)
    deq = dequantize_blockwise(codes, mins, scales, QWZ_BLOCK)
    return refresh_primary(deq, param_dtype)
