#!/usr/bin/env python3
"""Factor one workload on cuda:0 and time the PCG solve to 1e-8 (device ms),
twice (the first call also builds G rows / levels / tail). Prints one JSON line.
  python tools/pcg_time.py [--n 128] [--workload poisson3d]"""
import argparse, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2505_02977_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=128)
ap.add_argument("--workload", default="poisson3d")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mode", default="default", choices=["default", "exact", "fast"])
a = ap.parse_args()
g = {"poisson3d": lambda: P.gen_poisson3d(a.n), "poisson27": lambda: P.gen_poisson27(a.n, 1),
     "poisson2d": lambda: P.gen_poisson2d(a.n)}[a.workload]()
o = P.ordering_random(g.n, 0)
ctx = P.GpuContext(0)
f = P.factor_gpu(g, o, 0, ctx=ctx)
b = P.make_rhs(g, "random_projected", 0)
ctx.set_preconditioner_mode(a.mode)
res = []
for _ in range(a.reps):
    x, rep = P.rchol._pcg_resident(ctx, b, P.SolveConfig(tol=1e-8))
    res.append({"iters": rep.iterations, "relres": rep.relative_residual, "solve_ms": rep.device_ms,
                "wall_ms": rep.solve_seconds * 1e3, "exact": rep.exact})
print(json.dumps({"workload": a.workload, "n": a.n, "mode": a.mode, "tail_rows": os.environ.get("PARAC_TAIL_ROWS", "auto"),
                  "runs": res}))
