#!/usr/bin/env python
"""Summarize an `ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,
dram__bytes_read.sum,dram__bytes_write.sum` capture of tools/nvlink_bytes.py (one Falcon-7B
block, one step of P ranks driven from one process) into per-launch NVLink / DRAM bytes
next to their algorithmic counts, and (--traffic) merge the per-kernel means into
profiles/ncu_traffic.json, where bench.py reads the `roofline.traffic` of an N = P run.

    python tools/nvlink_summary.py CSV PLAIN_JSON OUT_JSON [--traffic profiles/ncu_traffic.json]

PLAIN_JSON = the line tools/nvlink_bytes.py printed (algorithmic bytes per launch).  The
captured launches are one step's: P forward gathers (device order), P backward gathers,
P fused RS+Adam."""
import argparse
import csv
import io
import json
from collections import OrderedDict


def parse(path):
    rows = [l for l in open(path) if l.startswith('"')]
    launches = OrderedDict()
    for r in csv.DictReader(io.StringIO("".join(rows))):
        x = launches.setdefault(r["ID"], {"kernel": r["Kernel Name"], "gpu": int(r["Device"]), "m": {}})
        x["m"][r["Metric Name"]] = (float(r["Metric Value"].replace(",", "")), r["Metric Unit"])
    return list(launches.values())


def to_bytes(v, unit):
    return v * {"byte": 1, "Kbyte": 1e3, "KB": 1e3, "Mbyte": 1e6, "MB": 1e6, "Gbyte": 1e9, "GB": 1e9}[unit]


def to_us(v, unit):
    return v * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}[unit]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("plain")
    ap.add_argument("out")
    ap.add_argument("--traffic", default=None)
    a = ap.parse_args()
    plain = json.loads([l for l in open(a.plain) if l.startswith("{")][-1])
    P, Pp = plain["world"], plain["node_size"]
    L = parse(a.csv)
    kinds, n_gather = [], 0
    for x in L:
        if "rs_tma" in x["kernel"]:
            kinds.append("reduce_scatter+adam")
        else:
            kinds.append("fwd_gather" if n_gather < P else "bwd_gather")
            n_gather += 1
    out = []
    for i, (x, k) in enumerate(zip(L, kinds)):
        m = x["m"]
        dur = to_us(*m["gpu__time_duration.sum"])
        rx, tx = to_bytes(*m["nvlrx__bytes.sum"]), to_bytes(*m["nvltx__bytes.sum"])
        dram = to_bytes(*m["dram__bytes_read.sum"]) + to_bytes(*m["dram__bytes_write.sum"])
        alg = plain["nvlink_ingress_alg_bytes_per_launch"][k][0]
        hbm = plain["local_hbm_alg_bytes_per_launch"][k][0]
        out.append({"launch": i, "gpu": x["gpu"], "kernel": k, "duration_us": round(dur, 1),
                    "nvlink_rx_bytes": int(rx), "nvlink_tx_bytes": int(tx), "alg_ingress_bytes": alg,
                    "rx_over_alg": round(rx / alg, 4) if alg else None,
                    "dram_bytes": int(dram), "local_hbm_alg_bytes": hbm, "dram_over_alg": round(dram / hbm, 4)})
    doc = {"what": f"ncu --metrics nvlrx__bytes.sum,nvltx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                   f"gpu__time_duration.sum of each hot kernel, one Falcon-7B block, world {P} (P'={Pp}), "
                   f"verify fingerprint, driven from ONE process (tools/nvlink_bytes.py) so ncu's serialization "
                   f"cannot deadlock; each profiled kernel runs ALONE (peers idle): the counters are its own "
                   f"traffic on its own GPU, the durations are single-puller rates, not the bench's all-to-all",
           "launches": out}
    json.dump(doc, open(a.out, "w"), indent=1)
    if a.traffic:
        tr = json.load(open(a.traffic))
        for k in ("fwd_gather", "bwd_gather", "reduce_scatter+adam"):
            xs = [o for o in out if o["kernel"] == k]
            if not xs:
                continue
            tr[f"P{P}_{k}"] = {
                "kernel": k, "world": P, "node_size": Pp, "captured_on": f"falcon7b_block, world {P} (P'={Pp}), one process driving {P} GPUs, "
                                          f"mean over the {len(xs)} GPUs' launches",
                "dram_bytes_per_launch": round(sum(o["dram_bytes"] for o in xs) / len(xs)),
                "launch_alg_bytes": xs[0]["local_hbm_alg_bytes"],
                "alg_bytes_are": "this GPU's own DRAM bytes (own slice / shard read, outputs written); peers' "
                                 "reads of this GPU's memory are counted in their own launches",
                "nvlink_rx_bytes_per_launch": round(sum(o["nvlink_rx_bytes"] for o in xs) / len(xs)),
                "nvlink_alg_ingress_bytes": xs[0]["alg_ingress_bytes"],
                "duration_us_standalone": round(sum(o["duration_us"] for o in xs) / len(xs), 1),
                "source": f"{a.out} (ncu --metrics ... --clock-control none, tools/nvlink_bytes.py --world {P} "
                          f"--node-size {Pp})"}
        json.dump(tr, open(a.traffic, "w"), indent=1)
    for o in out:
        print(o)


if __name__ == "__main__":
    main()
