#!/usr/bin/env python3
"""Aggregate ncu SASS stall samples per CUDA source line (cuda,sass view).
  python tools/ncu_lines.py report.ncu-rep [N] [--exclude stall_sleep,stall_barrier] [--file eliminate.cu] [--lines a-b]"""
import argparse, csv, io, subprocess, collections
ap = argparse.ArgumentParser()
ap.add_argument("rep"); ap.add_argument("n", nargs="?", type=int, default=30)
ap.add_argument("--exclude", default="stall_sleep")
ap.add_argument("--file", default=None)
ap.add_argument("--lines", default=None)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
excl = set(a.exclude.split(",")) if a.exclude else set()
hdr = None; cur = None; fpath = None
agg = collections.defaultdict(lambda: collections.Counter())
src = {}
for r in rows:
    if not r: continue
    if r[0] == "File Path": fpath = r[1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None: continue
    if r[0] and not r[0].isdigit(): continue
    if r[0]:  # source line
        cur = (fpath.split("/")[-1], int(r[0])); src[cur] = r[1]; continue
    if cur is None: continue
    for i, c in enumerate(hdr):
        if c.startswith("stall_") and "Not Issued" not in c and c not in excl and i < len(r) and r[i] not in ("", "-"):
            agg[cur][c] += float(r[i].replace(",", ""))
    ie = hdr.index("Instructions Executed")
    if ie < len(r) and r[ie] not in ("", "-"):
        agg[cur]["_exec"] += float(r[ie].replace(",", ""))
lo, hi = (map(int, a.lines.split("-")) if a.lines else (0, 10**9))
items = [(k, v) for k, v in agg.items() if (a.file is None or k[0] == a.file) and lo <= k[1] <= hi]
tot = sum(sum(x for kk, x in v.items() if kk != "_exec") for _, v in items)
print(f"samples (excluding {sorted(excl)}): {tot:.0f}")
for k, v in sorted(items, key=lambda kv: -sum(x for kk, x in kv[1].items() if kk != "_exec"))[:a.n]:
    s = sum(x for kk, x in v.items() if kk != "_exec")
    top = ", ".join(f"{kk[6:]}:{x:.0f}" for kk, x in v.most_common(4) if kk != "_exec")
    print(f"{k[0]}:{k[1]:<5d} {s / tot * 100:5.1f}% exec={v['_exec']:>10.0f} | {top} | {src.get(k, '').strip()[:70]}")
