#!/usr/bin/env python3
"""Median device times of the 64 x 64^3 batch (BASELINE config[4]) in one
context: python tools/batch_time.py [--c0 C] [--reps 3]"""
import argparse, json, os, statistics, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_02977_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--c0", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = P.gen_poisson3d(64)
gs = [g] * 64
os_ = [P.ordering_random(g.n, i) for i in range(64)]
ctx = P.GpuContext(0)
ms = []
for _ in range(a.reps + 1):
    fs, info = P.factor_batch_gpu(gs, os_, list(range(64)), P.GpuOptions(first_chunk=a.c0), ctx=ctx)
    ms.append((info.eliminate_ms, info.device_ms))
ms = ms[1:]
print(json.dumps({"c0": a.c0, "eliminate_ms": statistics.median(m[0] for m in ms),
                  "device_ms": statistics.median(m[1] for m in ms), "checksum0": f"{fs[0].checksum():016x}"}))
