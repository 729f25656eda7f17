#!/usr/bin/env python3
"""One 128^3 (or --n) factorization for ncu captures: warm-up run, then one
profiled run. Prints nothing measured (numbers under a profiler are not bench values)."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_02977_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--pcg", action="store_true")
a = ap.parse_args()
g = P.gen_poisson3d(a.n)
o = P.ordering_random(g.n, 0)
ctx = P.GpuContext(0)
f = P.factor_gpu(g, o, 0, ctx=ctx)
if a.pcg:
    b = P.make_rhs(g, "random_projected", 0)
    P.rchol._pcg_resident(ctx, b, P.SolveConfig(tol=1e-8))
print("done", f.checksum())
