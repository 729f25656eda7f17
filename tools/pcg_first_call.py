#!/usr/bin/env python3
"""First-call cost of the PCG on a new factor: process-first call (includes
CUDA lazy module loading of the solve kernels) vs a later call on a NEW factor
(layout build only) vs steady state. Prints one JSON line."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_02977_b200 as P

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
g = P.gen_poisson3d(n)
ctx = P.GpuContext(0)
b = P.make_rhs(g, "random_projected", 0)
out = {}
for seed in (0, 1):
    f = P.factor_gpu(g, P.ordering_random(g.n, seed), seed, ctx=ctx)
    t = time.perf_counter(); P.rchol._pcg_resident(ctx, b, P.SolveConfig(tol=1e-8)); t1 = time.perf_counter() - t
    t = time.perf_counter(); _, rep = P.rchol._pcg_resident(ctx, b, P.SolveConfig(tol=1e-8)); t2 = time.perf_counter() - t
    out[f"factor{seed}"] = {"first_ms": t1 * 1e3, "second_ms": t2 * 1e3, "device_ms": rep.device_ms}
print(json.dumps(out))
