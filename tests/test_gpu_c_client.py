"""The C ABI without Python: tests/c_abi/step_demo.c (C99 + the CUDA runtime only) runs
three training steps of two emulated ranks through libhpz.so on the GPU and checks the
gathers and the device counters itself."""
import os
import subprocess

import pytest

from .gpu_util import gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a GPU")]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def test_c_client_trains_through_the_abi(tmp_path):
    from paper_2407_01614_b200 import hpz as H
    libdir = os.path.dirname(H.LIB_PATH)
    exe = tmp_path / "step_demo"
    r = subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        "-I", os.path.join(CUDA, "include"), os.path.join(ROOT, "tests", "c_abi", "step_demo.c"),
                        "-L", libdir, "-lhpz", "-L", os.path.join(CUDA, "lib64"), "-lcudart",
                        f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{os.path.join(CUDA, 'lib64')}", "-o", str(exe)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "C_STEP_OK" in out.stdout, out.stdout + out.stderr
