#!/usr/bin/env python3
"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel
count / total / mean; optional --series NAME prints per-launch us of one kernel."""
import argparse, collections, csv
ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--series", default=None)
ap.add_argument("--top", type=int, default=15)
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
ks = [(r[ki], float(r[vi].replace(",", ""))) for r in rows[hdr + 1:] if len(r) > vi]
agg = collections.defaultdict(lambda: [0, 0.0])
for k, v in ks:
    key = k.split("(")[0].replace("(anonymous namespace)::", "")[:64]
    agg[key][0] += 1
    agg[key][1] += v
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:a.top]:
    print(f"{k:64s} {c:6d} {t / 1e6:9.2f} ms {t / c / 1e3:9.2f} us")
if a.series:
    s = [v for k, v in ks if a.series in k]
    print(len(s), [round(v / 1e3, 1) for v in s[:200]])
