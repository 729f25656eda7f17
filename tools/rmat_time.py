#!/usr/bin/env python3
"""Device factor time of an R-MAT graph (hub columns): python tools/rmat_time.py [--scale 20] [--reps 3]"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_02977_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = P.gen_rmat(a.scale, 16, 0)
o = P.ordering_random(g.n, 0)
ctx = P.GpuContext(0)
ms = []
for _ in range(a.reps + 1):
    st = P.FactorStats()
    f = P.factor_gpu(g, o, 0, P.GpuOptions(), st, ctx=ctx)
    ms.append(st.eliminate_ms)
print(json.dumps({"scale": a.scale, "eliminate_ms": statistics.median(ms[1:]), "all": ms,
                  "checksum": f"{f.checksum():016x}"}))
