#!/usr/bin/env python3
"""Per-kernel DRAM traffic and achieved HBM bandwidth from an ncu launch list
captured with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(--csv --log-file). Cold-cache, serialised launches: shares and bytes are
meaningful, absolute times are not bench values.
  python tools/kernel_hbm.py launches.csv [--out profiles/r01_kernel_hbm.csv] [--peak 6553.9]"""
import argparse, collections, csv
ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--out", default=None)
ap.add_argument("--peak", type=float, default=6553.9)
a = ap.parse_args()
rows = list(csv.reader(open(a.csv)))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9, "us": 1e-6,
         "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0}
per, names = collections.defaultdict(dict), {}
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    names[r[ii]] = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("void ", "")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    g = agg[names[i]]
    g[0] += 1
    g[1] += m.get("gpu__time_duration.sum", 0.0)
    g[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot_t = sum(v[1] for v in agg.values())
out = [(k, c, t, b) for k, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])]
lines = [["kernel", "launches", "mean_us", "share_of_time", "dram_MB_per_launch", "dram_GBps", f"frac_of_{a.peak}"]]
for k, c, t, b in out:
    gbs = b / t / 1e9 if t > 0 else 0.0
    lines.append([k, c, round(t / c * 1e6, 2), round(t / tot_t, 4), round(b / c / 1e6, 3), round(gbs, 1),
                  round(gbs / a.peak, 4)])
if a.out:
    csv.writer(open(a.out, "w")).writerows(lines)
for l in lines[:30]:
    print("  ".join(str(x)[:48].ljust(48 if i == 0 else 10) for i, x in enumerate(l)))
