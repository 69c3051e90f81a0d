"""Parity at BASELINE sizes in the bench's launch configuration (tests/full_size_worker.py):
Falcon-7B-shaped buffers (6.9e9 parameters), sampled elements vs the oracle."""
import os
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0
pytestmark = [pytest.mark.gpu, pytest.mark.skipif(NGPU < 1, reason="needs a GPU")]


def test_full_size_falcon7b_n1():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "full_size_worker.py")],
                         capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0 and "FULL_SIZE_OK" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_full_size_falcon7b_multiproc():
    n = 4 if NGPU >= 4 else 2
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port=30111", os.path.join(ROOT, "tests", "full_size_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert res.returncode == 0 and "FULL_SIZE_OK" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]


def test_full_size_block_eight_processes_sharing_gpus():
    """One full-size Falcon-7B decoder block (207M elements: every CTA wraps its ring many
    times) at the north_star's 2x4 topology, 8 separate processes on min(8, #GPUs) devices
    (a 1-GPU box included), sampled elements vs the oracle, in the bench's configuration."""
    env = dict(os.environ, HPZ_SHARE_GPUS="1", HPZ_FULL_MODEL="falcon7b_block")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=8",
           "--master-addr", "127.0.0.1", "--master-port=30131", os.path.join(ROOT, "tests", "full_size_worker.py")]
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert res.returncode == 0 and "FULL_SIZE_OK" in res.stdout, res.stdout[-2000:] + res.stderr[-2000:]
