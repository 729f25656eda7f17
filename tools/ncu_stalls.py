#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples in an ncu report (with source
correlation): python tools/ncu_stalls.py report.ncu-rep [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
ia, isrc, iall = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
iex = h.index("Instructions Executed")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
tot = sum(float(r[iall] or 0) for r in data if len(r) > iall)
print("total samples", tot)
for r in sorted(data, key=lambda r: -float(r[iall] or 0))[:N]:
    st = sorted(((float(r[i] or 0), h[i]) for i in stall_cols), reverse=True)[:2]
    print(f"{r[ia][-5:]} {float(r[iall]) / tot * 100:5.1f}% ex={r[iex]:>10} {r[isrc][:60]:60s} {st[0][1]}:{st[0][0]:.0f} {st[1][1]}:{st[1][0]:.0f}")
