"""Real multi-process path: one process per GPU, CUDA IPC peer mappings, NVLink P2P
pulls and cross-GPU release/acquire flags, checked against the oracle (tests/mp_worker.py).
Skipped unless the box has >= 2 GPUs (gpurun --gpus 2|4)."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu,
              pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")]


def _run(n, node_size, order="fixed", extra=(), port=29611):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mp_worker.py"), "--node-size", str(node_size), "--order", order, *extra]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert res.returncode == 0 and "MP_PARITY_OK" in res.stdout, res.stdout[-3000:] + res.stderr[-3000:]
    return res.stdout


@pytest.mark.parametrize("n,node", [(2, 1), (2, 2), (4, 2), (4, 1), (4, 4), (8, 4), (8, 2)])
def test_multiproc_parity_fixed(n, node):
    if n > NGPU:
        pytest.skip(f"needs {n} GPUs")
    _run(n, node, port=29611 + n * 10 + node)                       # TMA engine, fused RS+Adam


@pytest.mark.parametrize("n,node", [(2, 1), (4, 2), (8, 4)])
def test_multiproc_parity_ldg_exact_unfused(n, node):
    if n > NGPU:
        pytest.skip(f"needs {n} GPUs")
    _run(n, node, extra=("--engine", "ldg", "--verify", "exact", "--fused", "0"), port=29711 + n * 10 + node)


def test_multiproc_parity_off():
    _run(2, 1, order="off", port=29681)


def test_multiproc_stock_shows_mismatches():
    _run(2, 2, order="stock", extra=("--stock-delay-us", "3000"), port=29691)


@pytest.mark.parametrize("n,node", [(2, 1), (4, 2), (8, 4)])
def test_multiproc_parity_qgz(n, node):
    if n > NGPU:
        pytest.skip(f"needs {n} GPUs")
    _run(n, node, extra=("--qgz", "1"), port=29811 + n * 10 + node)


@pytest.mark.parametrize("n,node", [(2, 2), (4, 2)])
def test_multiproc_parity_bf16_grads(n, node):
    if n > NGPU:
        pytest.skip(f"needs {n} GPUs")
    _run(n, node, extra=("--grad-dtype", "bf16"), port=29911 + n * 10 + node)


@pytest.mark.parametrize("n,node", [(2, 1), (4, 2)])
def test_multiproc_parity_qwz_qgz(n, node):
    if n > NGPU:
        pytest.skip(f"needs {n} GPUs")
    _run(n, node, extra=("--qwz", "1", "--qgz", "1"), port=30011 + n * 10 + node)


def _mp_draw(seed):
    import numpy as np
    rng = np.random.default_rng(2000 + seed)
    n = int(rng.choice([2, 4]))
    node = int(rng.choice([d for d in (1, 2, 4) if d <= n and n % d == 0]))
    quant = str(rng.choice(["none", "qgz", "qwz", "both"]))
    qgz, qwz = quant in ("qgz", "both"), quant in ("qwz", "both")
    order = "fixed" if qwz else str(rng.choice(["fixed", "paper", "off"]))
    engine = str(rng.choice(["tma", "ldg"]))
    verify = "exact" if engine == "ldg" and not qwz and rng.random() < 0.5 else "fingerprint"
    numels = [int(x) for x in rng.integers(1, 400_000, 3)]
    extra = ["--engine", engine, "--verify", verify, "--fused", str(int(rng.random() < 0.6)),
             "--numels", ",".join(map(str, numels)), "--grad-slots", str(int(rng.integers(1, 4)))]
    if qgz:
        extra += ["--qgz", "1"]
    elif rng.random() < 0.3:
        extra += ["--grad-dtype", "bf16"]
    if qwz:
        extra += ["--qwz", "1"]
    return n, node, order, extra


@pytest.mark.parametrize("case", range(8))
def test_multiproc_fuzz_option_combinations(case):
    """Seeded random option combinations over real NVLink P2P (one process per GPU)."""
    n, node, order, extra = _mp_draw(case)
    if n > NGPU:
        pytest.skip(f"needs {n} GPUs")
    _run(n, node, order=order, extra=tuple(extra), port=30611 + case)
