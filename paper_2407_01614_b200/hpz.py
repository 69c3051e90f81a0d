"""Thin ctypes binding of libhpz.so (include/hpz.h).  Argument marshalling only:
every step of the hot path runs in the library's sm_100a kernels.  There is no
fallback: if the shared library is missing or fails to load, importing the
binding raises.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, byref, c_char_p, c_double, c_float, c_int, c_int64, c_uint64, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
# HPZ_LIB: another in-tree build of the same sources (A/B experiments, abtest_*/libhpz.so)
LIB_PATH = os.environ.get("HPZ_LIB") or os.path.join(_HERE, "libhpz.so")

HPZ_OK, HPZ_EINVAL, HPZ_ESTATE, HPZ_ECUDA, HPZ_ETIMEOUT, HPZ_ENOMEM = 0, -1, -2, -3, -4, -5
HPZ_F32, HPZ_BF16 = 0, 1
ORDER = {"fixed": 0, "stock": 1, "off": 2, "paper": 3}
VERIFY = {"none": 0, "fingerprint": 1, "exact": 2}
BUF = {"primary": 0, "master": 1, "m": 2, "v": 3, "grad_shard": 4, "secondary": 5, "grad_slot": 6}
IPC_HANDLE_BYTES = 64
MAX_WORLD = 16
STATUS_NAMES = {0: "HPZ_OK", -1: "HPZ_EINVAL", -2: "HPZ_ESTATE", -3: "HPZ_ECUDA", -4: "HPZ_ETIMEOUT", -5: "HPZ_ENOMEM"}

EXPORTED = [
    "hpz_init", "hpz_register_flat_params", "hpz_arena_alloc", "hpz_arena_open", "hpz_bind",
    "hpz_finalize", "hpz_layer_info", "hpz_arena_ptr", "hpz_buffer", "hpz_current_step",
    "hpz_counters", "hpz_last_error", "hpz_version", "hpz_set_order", "hpz_set_verify",
    "hpz_set_timeout", "hpz_load_master", "hpz_synth_master", "hpz_fwd_gather", "hpz_bwd_gather",
    "hpz_grad_buffer", "hpz_grad_upload", "hpz_synth_grads", "hpz_grads_ready",
    "hpz_reduce_scatter", "hpz_step", "hpz_reduce_scatter_adam", "hpz_set_option", "hpz_load_state",
    "hpz_resync_step", "hpz_secondary_copy",
]
OPT = {"store_grad_shard": 0, "ctas_per_sm": 1, "copy_engine": 2, "qgz": 3, "grad_dtype": 4, "qwz": 5, "max_ctas": 6,
       "bwd_ctas": 10, "rs_ctas": 11, "device_epoch": 13, "fault": 14,
       "alias_secondary": 15, "copy_by_caller": 16}
FAULT_SKIP_E1, FAULT_SKIP_E2 = 1, 2
COPY = {"ldg": 0, "tma": 1}


class hpz_adam(ctypes.Structure):
    _fields_ = [("lr", c_double), ("beta1", c_double), ("beta2", c_double), ("eps", c_double),
                ("weight_decay", c_double), ("step", c_int64)]


class hpz_layer_info_t(ctypes.Structure):
    _fields_ = [("numel", c_int64), ("numel_pad", c_int64), ("shard", c_int64), ("sec_shard", c_int64),
                ("off_primary", c_uint64), ("off_master", c_uint64), ("off_m", c_uint64), ("off_v", c_uint64),
                ("off_grad_shard", c_uint64), ("off_secondary", c_uint64), ("off_grad_slot", c_uint64),
                ("grad_slot", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class hpz_counters_t(ctypes.Structure):
    _fields_ = [("mismatches", c_uint64), ("nan_reads", c_uint64), ("fp_mismatches", c_uint64),
                ("fp_checked", c_uint64), ("timeouts", c_uint64), ("launches", c_uint64),
                ("fp_fwd_mismatches", c_uint64), ("fp_fwd_checked", c_uint64)]


class HpzError(RuntimeError):
    def __init__(self, fn: str, code: int, msg: str):
        super().__init__(f"{fn} -> {STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


def _load() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2407_01614_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = c_void_p
    sig = {
        "hpz_version": (c_int, []),
        "hpz_init": (c_int, [c_int, c_int, c_int, c_int, POINTER(c_void_p)]),
        "hpz_register_flat_params": (c_int, [P, c_int, POINTER(c_int64), c_int, c_int64, c_int, POINTER(c_uint64)]),
        "hpz_arena_alloc": (c_int, [P, c_void_p]),
        "hpz_arena_open": (c_int, [P, c_void_p]),
        "hpz_bind": (c_int, [P, POINTER(c_void_p)]),
        "hpz_finalize": (c_int, [P]),
        "hpz_layer_info": (c_int, [P, c_int, POINTER(hpz_layer_info_t)]),
        "hpz_arena_ptr": (c_int, [P, c_int, POINTER(c_void_p)]),
        "hpz_buffer": (c_int, [P, c_int, c_int, POINTER(c_void_p), POINTER(c_int64)]),
        "hpz_current_step": (c_int, [P, POINTER(c_int64)]),
        "hpz_resync_step": (c_int, [P]),
        "hpz_secondary_copy": (c_int, [P, c_int, c_void_p]),
        "hpz_counters": (c_int, [P, POINTER(hpz_counters_t), c_int]),
        "hpz_last_error": (c_char_p, [P]),
        "hpz_set_order": (c_int, [P, c_int, c_int, c_int]),
        "hpz_set_verify": (c_int, [P, c_int]),
        "hpz_set_timeout": (c_int, [P, c_double]),
        "hpz_load_master": (c_int, [P, c_int, c_void_p, c_void_p]),
        "hpz_synth_master": (c_int, [P, c_int, c_uint64, c_float, c_void_p]),
        "hpz_fwd_gather": (c_int, [P, c_int, c_void_p, c_void_p]),
        "hpz_bwd_gather": (c_int, [P, c_int, c_void_p, c_void_p]),
        "hpz_grad_buffer": (c_int, [P, c_int, POINTER(c_void_p), c_void_p]),
        "hpz_grad_upload": (c_int, [P, c_int, c_void_p, c_int64, c_void_p]),
        "hpz_synth_grads": (c_int, [P, c_int, c_uint64, c_float, c_int, c_void_p]),
        "hpz_grads_ready": (c_int, [P, c_int, c_void_p]),
        "hpz_reduce_scatter": (c_int, [P, c_int, c_void_p]),
        "hpz_step": (c_int, [P, c_int, POINTER(hpz_adam), c_void_p]),
        "hpz_reduce_scatter_adam": (c_int, [P, c_int, POINTER(hpz_adam), c_void_p]),
        "hpz_set_option": (c_int, [P, c_int, c_int64]),
        "hpz_load_state": (c_int, [P, c_int, c_void_p, c_void_p, c_void_p, c_int64, c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def _check(ctx, fn: str, rc: int):
    if rc != HPZ_OK:
        msg = LIB.hpz_last_error(ctx).decode() if ctx else ""
        raise HpzError(fn, rc, msg)


def _stream(s) -> c_void_p:
    """Accept a torch.cuda.Stream, a raw cudaStream_t int, or None (legacy default)."""
    if s is None:
        return c_void_p(0)
    if hasattr(s, "cuda_stream"):
        return c_void_p(s.cuda_stream)
    return c_void_p(int(s))


# ---------------------------------------------------------------- same names as the C ABI
def hpz_version() -> int:
    return LIB.hpz_version()


def hpz_init(world: int, node_size: int, rank: int, device: int) -> c_void_p:
    ctx = c_void_p()
    _check(None, "hpz_init", LIB.hpz_init(world, node_size, rank, device, byref(ctx)))
    return ctx


def hpz_register_flat_params(ctx, numels, param_dtype: int = HPZ_BF16, align_elems: int = 256,
                             n_grad_slots: int | None = None) -> int:
    arr = (c_int64 * len(numels))(*[int(n) for n in numels])
    out = c_uint64()
    slots = len(numels) if n_grad_slots is None else n_grad_slots
    _check(ctx, "hpz_register_flat_params",
           LIB.hpz_register_flat_params(ctx, len(numels), arr, param_dtype, align_elems, slots, byref(out)))
    return out.value


def hpz_arena_alloc(ctx) -> bytes:
    buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
    _check(ctx, "hpz_arena_alloc", LIB.hpz_arena_alloc(ctx, buf))
    return buf.raw


def hpz_arena_open(ctx, handles: list[bytes]):
    blob = b"".join(handles)
    buf = ctypes.create_string_buffer(blob, len(blob))
    _check(ctx, "hpz_arena_open", LIB.hpz_arena_open(ctx, buf))


def hpz_bind(ctx, ptrs: list[int]):
    arr = (c_void_p * len(ptrs))(*[c_void_p(int(p)) for p in ptrs])
    _check(ctx, "hpz_bind", LIB.hpz_bind(ctx, arr))


def hpz_finalize(ctx):
    _check(None, "hpz_finalize", LIB.hpz_finalize(ctx))


def hpz_layer_info(ctx, layer: int) -> hpz_layer_info_t:
    out = hpz_layer_info_t()
    _check(ctx, "hpz_layer_info", LIB.hpz_layer_info(ctx, layer, byref(out)))
    return out


def hpz_arena_ptr(ctx, rank: int) -> int:
    out = c_void_p()
    _check(ctx, "hpz_arena_ptr", LIB.hpz_arena_ptr(ctx, rank, byref(out)))
    return out.value


def hpz_buffer(ctx, layer: int, kind: str | int) -> tuple[int, int]:
    ptr, n = c_void_p(), c_int64()
    k = BUF[kind] if isinstance(kind, str) else kind
    _check(ctx, "hpz_buffer", LIB.hpz_buffer(ctx, layer, k, byref(ptr), byref(n)))
    return ptr.value, n.value


def hpz_current_step(ctx) -> int:
    t = c_int64()
    _check(ctx, "hpz_current_step", LIB.hpz_current_step(ctx, byref(t)))
    return t.value


def hpz_resync_step(ctx):
    _check(ctx, "hpz_resync_step", LIB.hpz_resync_step(ctx))


def hpz_counters(ctx, reset: bool = False) -> dict:
    out = hpz_counters_t()
    _check(ctx, "hpz_counters", LIB.hpz_counters(ctx, byref(out), int(reset)))
    return {f: getattr(out, f) for f, _ in hpz_counters_t._fields_}


def hpz_last_error(ctx) -> str:
    return LIB.hpz_last_error(ctx).decode()


def hpz_set_order(ctx, order: str | int, stock_delay_us: int = 0, stock_poison: bool = False):
    o = ORDER[order] if isinstance(order, str) else order
    _check(ctx, "hpz_set_order", LIB.hpz_set_order(ctx, o, int(stock_delay_us), int(stock_poison)))


def hpz_set_verify(ctx, mode: str | int):
    m = VERIFY[mode] if isinstance(mode, str) else mode
    _check(ctx, "hpz_set_verify", LIB.hpz_set_verify(ctx, m))


def hpz_set_timeout(ctx, seconds: float):
    _check(ctx, "hpz_set_timeout", LIB.hpz_set_timeout(ctx, float(seconds)))


def hpz_load_master(ctx, layer: int, full_fp32_ptr: int, stream=None):
    _check(ctx, "hpz_load_master", LIB.hpz_load_master(ctx, layer, c_void_p(full_fp32_ptr), _stream(stream)))


def hpz_synth_master(ctx, layer: int, key: int, scale: float, stream=None):
    _check(ctx, "hpz_synth_master", LIB.hpz_synth_master(ctx, layer, c_uint64(key), c_float(scale), _stream(stream)))


def hpz_fwd_gather(ctx, layer: int, full_out_ptr: int, stream=None):
    _check(ctx, "hpz_fwd_gather", LIB.hpz_fwd_gather(ctx, layer, c_void_p(full_out_ptr), _stream(stream)))


def hpz_secondary_copy(ctx, layer: int, stream=None):
    _check(ctx, "hpz_secondary_copy", LIB.hpz_secondary_copy(ctx, layer, _stream(stream)))


def hpz_bwd_gather(ctx, layer: int, full_out_ptr: int, stream=None):
    _check(ctx, "hpz_bwd_gather", LIB.hpz_bwd_gather(ctx, layer, c_void_p(full_out_ptr), _stream(stream)))


def hpz_grad_buffer(ctx, layer: int, stream=None) -> int:
    out = c_void_p()
    _check(ctx, "hpz_grad_buffer", LIB.hpz_grad_buffer(ctx, layer, byref(out), _stream(stream)))
    return out.value


def hpz_grad_upload(ctx, layer: int, src_ptr: int, n: int, stream=None):
    _check(ctx, "hpz_grad_upload", LIB.hpz_grad_upload(ctx, layer, c_void_p(src_ptr), c_int64(n), _stream(stream)))


def hpz_synth_grads(ctx, layer: int, key: int, scale: float, kind: int = 0, stream=None):
    _check(ctx, "hpz_synth_grads",
           LIB.hpz_synth_grads(ctx, layer, c_uint64(key), c_float(scale), kind, _stream(stream)))


def hpz_grads_ready(ctx, layer: int, stream=None):
    _check(ctx, "hpz_grads_ready", LIB.hpz_grads_ready(ctx, layer, _stream(stream)))


def hpz_reduce_scatter(ctx, layer: int, stream=None):
    _check(ctx, "hpz_reduce_scatter", LIB.hpz_reduce_scatter(ctx, layer, _stream(stream)))


def make_adam(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, step=0) -> hpz_adam:
    return hpz_adam(lr, beta1, beta2, eps, weight_decay, step)


def hpz_step(ctx, layer: int, adam: hpz_adam, stream=None):
    _check(ctx, "hpz_step", LIB.hpz_step(ctx, layer, byref(adam), _stream(stream)))


def hpz_reduce_scatter_adam(ctx, layer: int, adam: hpz_adam, stream=None):
    _check(ctx, "hpz_reduce_scatter_adam", LIB.hpz_reduce_scatter_adam(ctx, layer, byref(adam), _stream(stream)))


def hpz_set_option(ctx, option: str | int, value: int):
    o = OPT[option] if isinstance(option, str) else option
    _check(ctx, "hpz_set_option", LIB.hpz_set_option(ctx, o, c_int64(int(value))))


def hpz_load_state(ctx, layer: int, master_ptr: int, m_ptr: int, v_ptr: int, adam_steps_done: int, stream=None):
    _check(ctx, "hpz_load_state", LIB.hpz_load_state(ctx, layer, c_void_p(master_ptr), c_void_p(m_ptr),
                                                     c_void_p(v_ptr), c_int64(adam_steps_done), _stream(stream)))
