"""CPU checks of the C ABI (no GPU compute): the library loads, exports every symbol
include/hpz.h declares, validates arguments, and its layout (a1) agrees with the
oracle's independent layout on random inputs."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "hpz.h")).read()
    return sorted(set(re.findall(r"HPZ_API\s+(?:int|const char\*)\s+(hpz_\w+)\(", src)))


@pytest.fixture(scope="module")
def H():
    from paper_2407_01614_b200 import build
    build.build()
    from paper_2407_01614_b200 import hpz
    return hpz


def test_exports_every_declared_symbol(H):
    names = _declared()
    assert len(names) >= 20
    lib = ctypes.CDLL(H.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(H.EXPORTED) == names


def test_library_is_sm100a_only(H):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", H.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_no_gpu_init(H):
    assert H.hpz_version() == 1
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(H.HpzError) as e:
            H.hpz_init(1, 1, 0, 0)
        assert e.value.code == H.HPZ_EINVAL


def test_argument_validation(H):
    for args in [(0, 1, 0), (17, 1, 0), (8, 3, 0), (4, 8, 0), (4, 2, 4), (4, 2, -1)]:
        with pytest.raises(H.HpzError) as e:
            H.hpz_init(*args, -1)
        assert e.value.code == H.HPZ_EINVAL
    ctx = H.hpz_init(4, 2, 1, -1)
    try:
        with pytest.raises(H.HpzError):
            H.hpz_register_flat_params(ctx, [100], align_elems=100)       # not a power of two
        with pytest.raises(H.HpzError):
            H.hpz_register_flat_params(ctx, [0])
        with pytest.raises(H.HpzError):
            H.hpz_register_flat_params(ctx, [10, 10], n_grad_slots=3)
        H.hpz_register_flat_params(ctx, [100, 200])
        with pytest.raises(H.HpzError) as e:
            H.hpz_register_flat_params(ctx, [100])
        assert e.value.code == H.HPZ_ESTATE
        with pytest.raises(H.HpzError) as e:
            H.hpz_arena_alloc(ctx)
        assert e.value.code == H.HPZ_ESTATE
        with pytest.raises(H.HpzError) as e:
            H.hpz_fwd_gather(ctx, 0, 0x1000)
        assert e.value.code == H.HPZ_ESTATE
        with pytest.raises(H.HpzError):
            H.hpz_layer_info(ctx, 2)
    finally:
        H.hpz_finalize(ctx)


def test_layout_matches_oracle(H):
    """a1: the library's integer layout == the oracle's (independent code) on random cases."""
    from oracle import hpz_oracle as O
    rng = np.random.default_rng(5)
    for _ in range(60):
        Pp = int(rng.choice([1, 2, 4, 8]))
        P = Pp * int(rng.choice([1, 2, 4]))
        if P > 16:
            continue
        dtype = int(rng.choice([0, 1]))
        A = int(rng.choice([8, 16, 256, 1024])) if dtype == 1 else int(rng.choice([8, 256]))
        numels = [int(x) for x in rng.integers(1, 3_000_000, int(rng.integers(1, 6)))]
        ctx = H.hpz_init(P, Pp, int(rng.integers(0, P)), -1)
        try:
            arena = H.hpz_register_flat_params(ctx, numels, dtype, A)
            prev_end = 0
            for i, n in enumerate(numels):
                info = H.hpz_layer_info(ctx, i)
                lay = O.LayerLayout(n, P, Pp, A)
                assert (info.numel, info.numel_pad, info.shard, info.sec_shard) == \
                    (lay.numel, lay.numel_pad, lay.shard, lay.sec_shard)
                elem = 2 if dtype == 1 else 4
                bufs = [(info.off_primary, lay.shard * elem), (info.off_master, lay.shard * 4),
                        (info.off_m, lay.shard * 4), (info.off_v, lay.shard * 4),
                        (info.off_grad_shard, lay.shard * 4)]
                if P == Pp:      # secondary aliased to the primary
                    assert info.off_secondary == info.off_primary and info.sec_shard == info.shard
                else:
                    bufs.append((info.off_secondary, lay.sec_shard * elem))
                offs = sorted(bufs)
                for (o, sz) in offs:
                    assert o % 4096 == 0 and o >= prev_end     # aligned, non-overlapping
                    prev_end = o + sz
                assert info.grad_slot == i
            last = H.hpz_layer_info(ctx, len(numels) - 1)
            assert last.off_grad_slot + last.numel_pad * 4 <= arena
        finally:
            H.hpz_finalize(ctx)


def test_baseline_layout_numbers(H):
    ctx = H.hpz_init(8, 4, 0, -1)
    try:
        H.hpz_register_flat_params(ctx, [207070080], 1, 256)
        info = H.hpz_layer_info(ctx, 0)
        assert (info.numel_pad, info.shard, info.sec_shard) == (207071232, 25883904, 51767808)
    finally:
        H.hpz_finalize(ctx)


def test_options_host_only(H):
    ctx = H.hpz_init(8, 4, 0, -1)
    try:
        with pytest.raises(H.HpzError):
            H.hpz_set_option(ctx, "qgz", 8)                # only INT4
        with pytest.raises(H.HpzError):
            H.hpz_set_option(ctx, 99, 1)
        with pytest.raises(H.HpzError):
            H.hpz_set_option(ctx, "copy_engine", 7)
        H.hpz_set_option(ctx, "qgz", 4)
        a_q = H.hpz_register_flat_params(ctx, [1_000_000, 2048])
        with pytest.raises(H.HpzError) as e:                # sizes the arena: before register only
            H.hpz_set_option(ctx, "qgz", 0)
        assert e.value.code == H.HPZ_ESTATE
    finally:
        H.hpz_finalize(ctx)
    ctx = H.hpz_init(8, 4, 0, -1)
    try:
        a = H.hpz_register_flat_params(ctx, [1_000_000, 2048])
    finally:
        H.hpz_finalize(ctx)
    # qgZ adds int4 codes (N̂/2 B) + (min, scale) per 64 elements (N̂/8 B) per gradient slot
    assert a_q - a >= (1_001_472 + 2048) * 0.625 - 4 * 4096


def test_c_client_compiles_and_links(H, tmp_path):
    """include/hpz.h is plain C: a C99 program includes it, links libhpz.so and checks a layout."""
    import subprocess
    exe = tmp_path / "layout_check"
    src = os.path.join(ROOT, "tests", "c_abi", "layout_check.c")
    libdir = os.path.dirname(H.LIB_PATH)
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src,
                        "-L", libdir, "-lhpz", f"-Wl,-rpath,{libdir}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "numel_pad=207071232" in out.stdout


def test_secondary_aliased_at_full_node(H):
    """P' == P: the secondary is the primary — same arena offset, no extra bytes.
    qwZ keeps a separate secondary (it holds the dequantized weights)."""
    numels = [1_000_000, 4099]
    sizes = {}
    for P, Pp, qwz in [(4, 4, 0), (4, 2, 0), (4, 4, 1), (1, 1, 0)]:
        ctx = H.hpz_init(P, Pp, 0, -1)
        try:
            if qwz:
                H.hpz_set_option(ctx, "qwz", 8)
            sizes[(P, Pp, qwz)] = H.hpz_register_flat_params(ctx, numels)
            for i in range(len(numels)):
                info = H.hpz_layer_info(ctx, i)
                assert (info.off_secondary == info.off_primary) == (P == Pp and not qwz)
        finally:
            H.hpz_finalize(ctx)
    # (4,2) stores a secondary of N̂/2 bf16 elements per layer that (4,4) does not
    assert sizes[(4, 2, 0)] - sizes[(4, 4, 0)] >= (1_001_472 // 2) * 2


def test_quantized_options_need_block_aligned_shards(H):
    for opt, val in (("qgz", 4), ("qwz", 8)):
        ctx = H.hpz_init(4, 2, 0, -1)
        try:
            H.hpz_set_option(ctx, opt, val)
            with pytest.raises(H.HpzError) as e:
                H.hpz_register_flat_params(ctx, [100_000], 1, 64)
            assert e.value.code == H.HPZ_EINVAL
            H.hpz_register_flat_params(ctx, [100_000], 1, 256)
        finally:
            H.hpz_finalize(ctx)


def test_experiment_options_validation(H):
    """Grid caps: accepted ranges, rejected values, and they may change after registration
    (they size nothing); removed option numbers are rejected."""
    ctx = H.hpz_init(4, 2, 1, -1)
    try:
        H.hpz_register_flat_params(ctx, [100_000], 1, 256)
        for opt, good, bad in (("bwd_ctas", 48, -1), ("rs_ctas", 100, -5)):
            H.hpz_set_option(ctx, opt, good)
            H.hpz_set_option(ctx, opt, 0)
            with pytest.raises(H.HpzError) as e:
                H.hpz_set_option(ctx, opt, bad)
            assert e.value.code == H.HPZ_EINVAL
        for gone in (7, 8, 9, 12):   # push gather / split phases / push RS / emulated inter-node link
            with pytest.raises(H.HpzError) as e:
                H.hpz_set_option(ctx, gone, 1)
            assert e.value.code == H.HPZ_EINVAL
    finally:
        H.hpz_finalize(ctx)
