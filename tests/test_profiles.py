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
