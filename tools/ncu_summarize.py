#!/usr/bin/env python3
"""Fold one `ncu --set full` capture (.ncu-rep) into profiles/ncu_summary.json.

  python tools/ncu_summarize.py gpurun_out/k3_full.ncu-rep --workload poisson3d_128 \
      --kernel eliminate_kernel --algorithmic-bytes 1347503868

Stores, per workload and kernel: duration, DRAM bytes read/written (the
`traffic` that bench.py reports), DRAM/L2/SM throughput percentages, issue
activity and occupancy. Numbers taken under ncu are evidence, never bench values.
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

KEYS = {
    "gpu__time_duration.sum": "duration_s",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "lts__t_bytes.sum": "l2_bytes",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__grid_size": "grid",
    "launch__registers_per_thread": "regs",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for name, unit, val in zip(head, units, r):
            if name in KEYS:
                try:
                    x = float(val.replace(",", ""))
                except ValueError:
                    continue
                d[KEYS[name]] = x * SCALE.get(unit, 1.0) if unit in SCALE else x
        d["kernel"] = r[head.index("Kernel Name")].split("(")[0]
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--kernel", required=True)
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_summary.json"))
    a = ap.parse_args()
    recs = [r for r in read_raw(a.rep) if a.kernel in r["kernel"]]
    if not recs:
        raise SystemExit(f"no {a.kernel} launch in {a.rep}")
    r = recs[0]
    r["dram_bytes"] = r.get("dram_read", 0) + r.get("dram_write", 0)
    if a.algorithmic_bytes:
        r["algorithmic_bytes"] = a.algorithmic_bytes
        r["traffic_over_algorithmic"] = r["dram_bytes"] / a.algorithmic_bytes
    r["source"] = os.path.basename(a.rep)
    summ = {}
    if os.path.exists(a.out):
        with open(a.out) as fh:
            summ = json.load(fh)
    w = summ.setdefault(a.workload, {})
    w[a.kernel] = r
    if a.kernel == "eliminate_kernel":
        w["eliminate_kernel_dram_bytes"] = r["dram_bytes"]
    with open(a.out, "w") as fh:
        json.dump(summ, fh, indent=1, sort_keys=True)
    print(json.dumps(r, indent=1))


if __name__ == "__main__":
    main()
