#!/usr/bin/env python3
"""Median device times of repeated factorizations of one staged graph
(setup / eliminate / after-K3 / device total, ms): A/B of environment knobs.

  python tools/factor_time.py [--workload poisson3d] [--n 128] [--reps 7]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_02977_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="poisson3d")
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--grid", type=int, default=0)
ap.add_argument("--c0", type=int, default=0)
a = ap.parse_args()
g = {"poisson3d": lambda: P.gen_poisson3d(a.n), "poisson27": lambda: P.gen_poisson27(a.n, 1),
     "poisson2d": lambda: P.gen_poisson2d(a.n), "rmat": lambda: P.gen_rmat(a.n, 16, 0)}[a.workload]()
ctx = P.GpuContext(0)
ctx.upload(g, P.ordering_random(g.n, 0))
rows = []
for _ in range(a.reps + 2):
    i = ctx.factor_resident(0, P.GpuOptions(grid_ctas=a.grid, first_chunk=a.c0))
    rows.append((i.setup_ms, i.eliminate_ms, i.assemble_ms, i.device_ms))
rows = rows[2:]
med = [statistics.median(r[j] for r in rows) for j in range(4)]
print(json.dumps({"workload": f"{a.workload}_{a.n}", "grid": a.grid, "c0": a.c0, "setup_ms": med[0], "eliminate_ms": med[1],
                  "after_k3_ms": med[2], "device_ms": med[3], "env": {k: v for k, v in os.environ.items()
                                                                      if k.startswith("PARAC_")}}))
