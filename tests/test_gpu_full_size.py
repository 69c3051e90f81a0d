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
