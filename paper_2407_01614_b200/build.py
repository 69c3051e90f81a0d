"""Build libhpz.so in-tree for sm_100a (nvcc; no torch extension machinery).

    python -m paper_2407_01614_b200.build          # or __graft_entry__.build()
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libhpz.so")
SOURCES = ["hpz_kernels.cu", "hpz_tma.cu", "hpz_runtime.cpp"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "hpz.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--shared", "-Xcompiler", "-fPIC",
           "-Xcompiler", "-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
           "-Xptxas", "-v" if verbose else "-O3",
           "-o", LIB + ".tmp"] + [os.path.join(CSRC, s) for s in SOURCES]
    # exported C ABI: hidden visibility by default, extern "C" functions re-exported below
    cmd += ["-Xcompiler", "-Wall"] + os.environ.get("HPZ_NVCC_FLAGS", "").split()
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libhpz.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(LIB + ".tmp", LIB)
    # design-experiment tool (not linked into the library): NVLink P2P strategy probe
    probe = os.path.join(ROOT, "tools", "p2p_probe.cu")
    if os.path.exists(probe):
        subprocess.run([NVCC, *ARCH, "-O3", "-o", os.path.join(ROOT, "tools", "p2p_probe"), probe],
                       capture_output=True, text=True)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
