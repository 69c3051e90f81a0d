#!/usr/bin/env python
"""Summarise an `ncu --set full` capture of the N=1 hot kernels (one Falcon-7B decoder block:
fwd gather, bwd gather, fused RS+Adam) into a per-kernel CSV under profiles/ and the
per-launch DRAM traffic bench.py reports as roofline.traffic (profiles/ncu_traffic.json).

    python tools/ncu_summary.py gpurun_out/r02_prof_n1.ncu-rep profiles/r02_ncu_full_n1.csv
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REP = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "prof_n1.ncu-rep")
OUT = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", "r02_ncu_full_n1.csv")
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]

from paper_2407_01614_b200 import shapes  # noqa: E402

numel = shapes.numels("falcon7b_block")[0]
npad = (numel + 255) // 256 * 256           # P = 1, A = 256
# algorithmic HBM bytes per launch at P = P' = 1 (secondary aliased to the primary, R29):
# gathers read the primary and write the full buffer; RS+Adam reads the gradient slot 4 +
# w, m, v 12 and writes w, m, v 12 + the bf16 primary 2
alg = {"fwd_gather": 4 * npad, "bwd_gather": 4 * npad, "reduce_scatter+adam": 30 * npad}
raw = subprocess.run(["ncu", "-i", REP, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units = rows[0], rows[1]
col = {k: h.index(k) for k in ("Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                               "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active")}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
tscale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}
out, traffic, gathers = [], {}, 0
src = os.path.relpath(OUT, ROOT)
for r in rows[2:]:
    name = r[col["Kernel Name"]]
    if "rs_tma_kernel" in name:
        kind = "reduce_scatter+adam"
    elif "gather_tma_kernel" in name:
        kind = "fwd_gather" if gathers == 0 else "bwd_gather"
        gathers += 1
    else:
        continue
    t = float(r[col["gpu__time_duration.sum"]]) * tscale[units[col["gpu__time_duration.sum"]]]
    rd = float(r[col["dram__bytes_read.sum"]]) * scale[units[col["dram__bytes_read.sum"]]]
    wr = float(r[col["dram__bytes_write.sum"]]) * scale[units[col["dram__bytes_write.sum"]]]
    ach = alg[kind] / t / 1e9
    out.append([kind, name, round(t * 1e6, 3), round(rd / 1e9, 4), round(wr / 1e9, 4), round((rd + wr) / 1e9, 4),
                round(alg[kind] / 1e9, 4), round(ach, 1), round(ach / PEAK, 4), r[col["launch__registers_per_thread"]],
                r[col["sm__warps_active.avg.pct_of_peak_sustained_active"]]])
    traffic[f"P1_{kind}"] = {"kernel": name, "captured_on": f"falcon7b_block ({npad:,} padded elements), N=1",
                             "dram_bytes_per_launch": rd + wr, "launch_alg_bytes": alg[kind],
                             "duration_us": round(t * 1e6, 3),
                             "source": f"{src} (ncu --set full --clock-control none)"}
with open(OUT, "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["# ncu --set full --clock-control none: one launch each, Falcon-7B decoder "
                f"block ({npad} padded elements), N=1; peak = MEASURED_PEAKS hbm_gbs {PEAK}"])
    w.writerow(["kernel", "name", "duration_us", "dram_read_GB", "dram_write_GB", "dram_total_GB", "algorithmic_GB",
                "achieved_GBps", "frac_of_hbm_peak", "registers", "warps_active_pct"])
    w.writerows(out)
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
for o in out:
    print(o)
