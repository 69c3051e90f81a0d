"""Seeded synthetic input generators shared by the oracle, the tests and the bench.

This module holds NONE of the method's arithmetic (no gathering, no reduction,
no optimizer): it only turns (seed, layer, step, rank, element index) into a
deterministic fp32 value.  The CUDA side implements the same counter-based
generator independently (``hpz_synth_*`` in csrc/hpz_kernels.cu); a GPU test
checks the two agree bit for bit.  See DESIGN.md "Input recipe".

Generator (integer only, no transcendentals, exact in fp32):

    mix(z)      = splitmix64 finaliser:  z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
                                          z ^= z>>27; z *= 0x94D049BB133111EB;
                                          z ^= z>>31            (all mod 2^64)
    key         = mix(mix(mix(mix(seed) ^ layer) ^ step) ^ rank)
    x(e)        = mix(key + (e + 1) * 0x9E3779B97F4A7C15)
    uniform(e)  = (int(x >> 40) - 2^23) * 2^-23 * scale      in [-scale, scale)
    dyadic(e)   = (int(x >> 53) - 2^10) * 2^-20              integers on a 2^-20 grid

``scale`` must be a power of two so every value is an exact fp32 number.
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
C1 = 0xBF58476D1CE4E5B9
C2 = 0x94D049BB133111EB

SEED_PARAMS = 0x5EED0001
SEED_GRADS = 0x5EED0002
SEED_TOY_DATA = 7
PARAM_SCALE = 2.0 ** -5
GRAD_SCALE = 2.0 ** -12


def mix_int(z: int) -> int:
    """splitmix64 finaliser on a Python int (host-side key derivation)."""
    z &= M64
    z ^= z >> 30
    z = (z * C1) & M64
    z ^= z >> 27
    z = (z * C2) & M64
    z ^= z >> 31
    return z


def stream_key(seed: int, layer: int, step: int, rank: int) -> int:
    """64-bit key of one (seed, layer, step, rank) stream; passed to the GPU as-is."""
    k = mix_int(seed)
    k = mix_int(k ^ (layer & M64))
    k = mix_int(k ^ (step & M64))
    k = mix_int(k ^ (rank & M64))
    return k


def _mix_arr(z: np.ndarray) -> np.ndarray:
    z = z ^ (z >> np.uint64(30))
    z = z * np.uint64(C1)
    z = z ^ (z >> np.uint64(27))
    z = z * np.uint64(C2)
    z = z ^ (z >> np.uint64(31))
    return z


def _raw(key: int, idx: np.ndarray) -> np.ndarray:
    e = np.asarray(idx, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(key) + (e + np.uint64(1)) * np.uint64(GOLDEN)
        return _mix_arr(z)


def uniform(key: int, idx, scale: float) -> np.ndarray:
    """fp32 values in [-scale, scale) on a 2^-23*scale grid (exact)."""
    x = _raw(key, idx)
    i = (x >> np.uint64(40)).astype(np.int64) - (1 << 23)
    return (i.astype(np.float64) * (2.0 ** -23) * scale).astype(np.float32)


def dyadic(key: int, idx) -> np.ndarray:
    """fp32 integers in [-2^10, 2^10) times 2^-20: every sum of <= 2^13 of them is exact."""
    x = _raw(key, idx)
    i = (x >> np.uint64(53)).astype(np.int64) - (1 << 10)
    return (i.astype(np.float64) * (2.0 ** -20)).astype(np.float32)


def layer_params(layer: int, numel: int, numel_pad: int | None = None,
                 seed: int = SEED_PARAMS, scale: float = PARAM_SCALE) -> np.ndarray:
    """Initial full fp32 parameters W0 of one flat layer buffer; zeros in padding."""
    n_pad = numel if numel_pad is None else numel_pad
    out = np.zeros(n_pad, dtype=np.float32)
    out[:numel] = uniform(stream_key(seed, layer, 0, 0), np.arange(numel), scale)
    return out


def layer_grads(layer: int, step: int, rank: int, numel: int, numel_pad: int | None = None,
                seed: int = SEED_GRADS, scale: float = GRAD_SCALE, kind: str = "uniform") -> np.ndarray:
    """Full-length synthetic gradient of rank ``rank`` for one layer at one step; zero padding."""
    n_pad = numel if numel_pad is None else numel_pad
    out = np.zeros(n_pad, dtype=np.float32)
    key = stream_key(seed, layer, step, rank)
    if kind == "uniform":
        out[:numel] = uniform(key, np.arange(numel), scale)
    elif kind == "dyadic":
        out[:numel] = dyadic(key, np.arange(numel))
    else:
        raise ValueError(kind)
    return out


def values_at(seed: int, layer: int, step: int, rank: int, idx, scale: float,
              numel: int) -> np.ndarray:
    """Generator values at sampled element indices (zero where idx >= numel)."""
    idx = np.asarray(idx, dtype=np.int64)
    v = uniform(stream_key(seed, layer, step, rank), idx, scale)
    v[idx >= numel] = 0.0
    return v
