"""The committed evidence is reproducible from the committed raw captures: the per-launch
NVLink / DRAM figures bench.py reads from profiles/ncu_traffic.json (roofline.traffic at
N = 2, 4) are what tools/nvlink_summary.py derives from the ncu CSVs, and every captured
kernel's DRAM traffic is within its algorithmic bytes (no wasted re-reads)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = lambda *a: os.path.join(ROOT, "profiles", *a)  # noqa: E731


@pytest.mark.parametrize("n", [2, 4])
def test_traffic_table_matches_ncu_capture(n, tmp_path):
    committed = json.load(open(P("ncu_traffic.json")))
    base = {k: v for k, v in committed.items() if not k.startswith(f"P{n}_")}
    tr = tmp_path / "traffic.json"
    tr.write_text(json.dumps(base))
    out = tmp_path / "summary.json"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "nvlink_summary.py"), P(f"r02_ncu_nvlink_n{n}.csv"),
                        P(f"r02_nvlink_plain_n{n}.json"), str(out), "--traffic", str(tr)],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    got = json.load(open(tr))
    for k in ("fwd_gather", "bwd_gather", "reduce_scatter+adam"):
        a, b = got[f"P{n}_{k}"], committed[f"P{n}_{k}"]
        for f in ("dram_bytes_per_launch", "launch_alg_bytes", "nvlink_rx_bytes_per_launch", "nvlink_alg_ingress_bytes"):
            assert a[f] == b[f], (k, f)
        assert a["dram_bytes_per_launch"] <= 1.0 * a["launch_alg_bytes"], k          # no re-reads
        if a["nvlink_alg_ingress_bytes"]:
            assert abs(a["nvlink_rx_bytes_per_launch"] / a["nvlink_alg_ingress_bytes"] - 1.125) < 0.01, k


def test_n1_traffic_within_algorithmic_bytes():
    t = json.load(open(P("ncu_traffic.json")))
    for k in ("P1_fwd_gather", "P1_bwd_gather", "P1_reduce_scatter+adam"):
        assert t[k]["dram_bytes_per_launch"] <= t[k]["launch_alg_bytes"], k


def test_bench_algorithmic_bytes_match_survey_c2():
    """bench.step_bytes (the roofline's and the per-kernel table's denominators) on the C2
    configuration — Falcon-7B, P = 8, P' = 4 and 2, layout from the ORACLE (independent of
    the library) — reproduces SURVEY §8's per-step figures: forward-gather ingress 12.11 GB
    (a2), backward 10.38 / 6.92 GB (a4), RS 24.23 GB (a5), fused Adam 25.96 GB of HBM (a6)."""
    sys.path.insert(0, ROOT)
    import bench
    from oracle import hpz_oracle as O
    from paper_2407_01614_b200 import shapes
    numels = shapes.numels("falcon7b")
    for Pp, bwd in ((4, 10.38), (2, 6.92)):
        lays = [O.LayerLayout(n, 8, Pp, 256) for n in numels]
        B = bench.step_bytes([x.numel_pad for x in lays], [x.shard for x in lays], 8, Pp, 2)
        assert round(B["nvlink"]["fwd_gather"] / 1e9, 2) == 12.11
        assert round(B["nvlink"]["bwd_gather"] / 1e9, 2) == bwd
        assert round(B["nvlink"]["reduce_scatter+adam"] / 1e9, 2) == 24.23
        assert round(B["adam"] / 1e9, 2) == 25.96
        # per padded element: 2(P-1)/P, 2(P'-1)/P', 4(P-1)/P, 30/P
        N = sum(x.numel_pad for x in lays)
        assert B["nvlink"]["fwd_gather"] == N * 2 * 7 / 8 and B["nvlink"]["bwd_gather"] == N * 2 * (Pp - 1) / Pp
        assert B["hbm_p1"]["reduce_scatter+adam"] == sum(x.shard for x in lays) * 30
    # P' = P: no secondary bytes; qwZ keeps one
    lays = [O.LayerLayout(n, 4, 4, 256) for n in numels]
    assert bench.step_bytes([x.numel_pad for x in lays], [x.shard for x in lays], 4, 4, 2)["sec"] == 0
    assert bench.step_bytes([x.numel_pad for x in lays], [x.shard for x in lays], 4, 4, 2, qwz=True)["sec"] > 0
