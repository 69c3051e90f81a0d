"""Separate processes per rank on however many GPUs the box has (one is enough): rank r runs
on GPU r % device_count, so on the driver's 1-GPU box every rank is its own process on
the same device.  Each process owns its arena (libhpz), maps its peers' arenas through
CUDA IPC and synchronizes with them only through the device-side release/acquire flags
(E1-E7) — the DistWorld path of one-process-per-GPU training, with the kernels of
different ranks genuinely concurrent (time-sliced contexts on a shared GPU, truly
parallel across GPUs).  Unlike EmulatedWorld (one process, one stream), no rank can
rely on another rank's release having been issued earlier in its own stream.

Every rank checks its own fwd / bwd gathers, secondary, RS and master / m / v / primary
bitwise against the CPU oracle (tests/mp_worker.py)."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(NGPU < 1, reason="needs a GPU")]


def _run(n, node_size, extra=(), port=31011):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mp_worker.py"), "--node-size", str(node_size), "--share-gpus", "1",
           "--steps", "2", *extra]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=420, cwd=ROOT)
    assert res.returncode == 0 and "MP_PARITY_OK" in res.stdout, res.stdout[-3000:] + res.stderr[-3000:]
    assert "timeouts=0" in res.stdout
    return res.stdout


@pytest.mark.parametrize("n,node", [(2, 1), (4, 2), (8, 4)])
def test_processes_sharing_gpus_parity(n, node):
    """P processes (8 = the north_star's 2x4 topology) on min(P, #GPUs) devices."""
    _run(n, node, port=31011 + n * 10 + node)


def test_processes_sharing_gpus_qgz_full_node():
    """qgZ reduce-scatter with P' = P (aliased secondary, E7) across processes."""
    _run(4, 4, extra=("--qgz", "1"), port=31111)


@pytest.mark.parametrize("n,node", [(8, 4), (8, 2)])
def test_bench_eight_ranks_sharing_gpus(n, node):
    """The driver's 8-GPU bench command path (self-launch of 8 ranks, DistWorld, device
    epochs + CUDA-graph capture of the step, fingerprint checks, the JSON line) on a box with
    fewer GPUs: `--share-gpus` puts the ranks on GPU r % device_count.  Functional only —
    the timings of time-sliced ranks are not measurements (the line says so)."""
    import json
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--node-size", str(node),
           "--share-gpus", "--model", "falcon7b_block", "--steps", "2", "--warmup", "3",
           "--no-cpu-baseline", "--no-e2e"]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stdout[-2000:] + res.stderr[-4000:]
    lines = [x for x in res.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, res.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["config"]["world"] == n and d["config"]["node_size"] == node
    assert "FUNCTIONAL CHECK" in d["config"]["share_gpus"]
    assert d["config"]["launch"].startswith("one step captured in a CUDA graph")
    st = d["stale_param_mismatches"]
    assert st["timeouts"] == 0 and st["fingerprint_layers"] == 0 and st["fwd_vs_owner_fingerprint_layers"] == 0
    assert st["layers_checked"] == n * 2 and st["fwd_layers_checked"] == n * 2
    assert d["gpu_launches"] > 0
