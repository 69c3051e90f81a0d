#!/usr/bin/env python
"""Tabulate tools/model_sweep.sh output (gpurun_out/sweep_*.json) as markdown + one JSON."""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out")
rows = []
for f in sorted(glob.glob(os.path.join(src, "sweep_*_n*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    b = d["breakdown_ms_per_step"]
    nc = d.get("nccl_baseline") or {}
    ncms = nc.get("ms_per_step") or {}
    rows.append({
        "model": os.path.basename(f).split("sweep_")[1].rsplit("_n", 1)[0], "n": d["n_gpus"],
        "P'": d["config"]["node_size"], "params": d["config"]["workload"].split("(")[1].split(")")[0],
        "step_ms": d["ms_per_step"], "fwd_ag_ms": b["fwd_gather"], "bwd_ag_ms": b["bwd_gather"],
        "rs_adam_ms": b["reduce_scatter+adam"], "grad_synth_ms": b.get("grad_synth", 0.0),
        "value_GBps": d["value"], "nvlink_GBps_per_gpu": d.get("nvlink_ingress_GBps_per_gpu"),
        "nvlink_frac_of_900": d.get("nvlink_frac_of_900"),
        "roofline": f'{d["roofline"]["kernel"]} {d["roofline"]["frac"]:.2f} of {d["roofline"]["peak"]} {d["roofline"]["unit"]}',
        "nccl_collectives_ms": round(sum(ncms.values()), 2) if ncms else None,
        "stale": d["stale_param_mismatches"]["fingerprint_layers"], "timeouts": d["stale_param_mismatches"]["timeouts"],
    })
order = {"falcon7b": 0, "llama2_7b": 1, "llama2_13b": 2, "falcon40b_block": 3, "llama2_70b_layers": 4}
rows.sort(key=lambda r: (order.get(r["model"], 9), r["n"]))
cols = ["model", "n", "P'", "step_ms", "fwd_ag_ms", "bwd_ag_ms", "rs_adam_ms", "grad_synth_ms", "value_GBps",
        "nvlink_GBps_per_gpu", "nvlink_frac_of_900", "roofline", "nccl_collectives_ms", "stale"]
print("| " + " | ".join(cols) + " |")
print("|" + "---|" * len(cols))
for r in rows:
    print("| " + " | ".join(str(r[c]) for c in cols) + " |")
json.dump(rows, open(os.path.join(ROOT, "profiles", "r01_model_sweep.json"), "w"), indent=1)
