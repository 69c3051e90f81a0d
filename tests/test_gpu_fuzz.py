"""Randomized option combinations vs the oracle (single-GPU rank emulation).

Each case draws a world (P, P'), layer sizes (incl. layers smaller than P*A and ragged
tails), parameter dtype, alignment and a legal combination of the options — copy engine,
verification, fused RS+Adam, ordering (fixed / paper / off), bf16 or qgZ gradients, qwZ,
shared gradient slots — then checks two steps
element by element with the same bars as test_gpu_parity (gathers, secondaries, RS,
master/m/v, primaries bit-exact).  Seeded: the cases are the same every run."""
import numpy as np
import pytest

from .gpu_util import ParityRun, gpu_ok
from .test_gpu_parity import _check_step

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a GPU")]

N_CASES = 128


def _draw(seed):
    rng = np.random.default_rng(1000 + seed)
    P = int(rng.choice([1, 2, 3, 4, 5, 6, 8]))
    Pp = int(rng.choice([d for d in range(1, P + 1) if P % d == 0]))
    dtype = str(rng.choice(["bf16", "f32"]))
    quant = str(rng.choice(["none", "none", "qgz", "qwz", "both"]))
    qgz, qwz = quant in ("qgz", "both"), quant in ("qwz", "both")
    align = 256 if (qgz or qwz) else int(rng.choice([8, 64, 256]))
    numels = [int(x) for x in rng.integers(1, 120_000, int(rng.integers(1, 5)))]
    engine = str(rng.choice(["tma", "ldg"]))
    verify = "exact" if engine == "ldg" and not qwz and rng.random() < 0.5 else \
        str(rng.choice(["fingerprint", "none"]))
    order = "fixed" if qwz else str(rng.choice(["fixed", "fixed", "paper", "off"]))
    grad_dtype = "bf16" if (not qgz and rng.random() < 0.3) else "f32"
    fused = bool(rng.random() < 0.6)
    slots = int(rng.integers(1, len(numels) + 1))
    return dict(numels=numels, world=P, node_size=Pp, dtype=dtype, align=align, copy_engine=engine,
                verify=verify, order=order, grad_dtype=grad_dtype, qgz=qgz, qwz=qwz,
                fused=fused, n_grad_slots=slots)


@pytest.mark.parametrize("case", range(N_CASES))
def test_fuzz_option_combinations(case):
    cfg = _draw(case)
    numels = cfg.pop("numels")
    P, Pp = cfg.pop("world"), cfg.pop("node_size")
    run = ParityRun(numels, P, Pp, **cfg)
    try:
        for _ in range(2):
            _check_step(run, run.step())
        c = run.counters()
        assert c["timeouts"] == 0, cfg
        assert c["fp_mismatches"] == 0 and c["mismatches"] == 0 and c["nan_reads"] == 0, cfg
    finally:
        run.close()
