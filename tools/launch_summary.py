#!/usr/bin/env python3
"""Summarise an `ncu --metrics gpu__time_duration.sum --csv --log-file X` launch list:
per-kernel launch count, total and mean device time (cold-cache, serialised)."""
import csv
import sys


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(r[ui], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    return agg


if __name__ == "__main__":
    agg = load(sys.argv[1])
    total = sum(v[1] for v in agg.values())
    print(f"{'kernel':34s} {'launches':>8s} {'total ms':>10s} {'mean us':>10s} {'share':>6s}")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} {c:8d} {t:10.3f} {1e3 * t / c:10.1f} {100 * t / total:5.1f}%")
    print(f"{'TOTAL':34s} {sum(v[0] for v in agg.values()):8d} {total:10.3f}")
