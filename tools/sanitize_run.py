#!/usr/bin/env python3
"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck): factor + PCG at 10^3, a 3-problem batch, an R-MAT graph whose hubs
take the cooperative hub path (with helpers, and with the owner alone on a
2-CTA grid), each checked against the oracle's checksum.
  compute-sanitizer --tool memcheck python tools/sanitize_run.py"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle
import paper_2505_02977_b200 as P

opts = P.GpuOptions(watchdog_seconds=1200.0)
ctx = P.GpuContext(0)
port = oracle.Port()


def check(g, perm, seed, f):
    want = port.factor(g, perm, seed)
    ref = P.LdlFactor(want["n"], want["col_ptr"], want["rows"], want["values"], want["diag"], want["perm"])
    assert f.same_values(ref), "factor differs from the oracle"


g = P.gen_poisson3d(10)
o = P.ordering_random(g.n, 1)
f = P.factor_gpu(g, o, 1, opts, ctx=ctx)
check(g, o.perm, 1, f)
b = P.make_rhs(g, "random_projected", 1)
x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=ctx)
assert rep.converged, rep
z = P.apply_preconditioner_gpu(f, b, ctx=ctx)
print("poisson 10^3 ok, pcg", rep.iterations)
gs = [P.gen_poisson3d(6), P.gen_poisson3d(7), P.gen_poisson2d(12)]
os_ = [P.ordering_random(x.n, i) for i, x in enumerate(gs)]
fs, _ = P.factor_batch_gpu(gs, os_, [0, 1, 2], ctx=ctx)
for i, (gg, oo, ff) in enumerate(zip(gs, os_, fs)):
    check(gg, oo.perm, i, ff)
print("batch ok")
g = P.gen_rmat(12, 16, 0)
o = P.ordering_random(g.n, 0)
f = P.factor_gpu(g, o, 0, opts, ctx=ctx)
check(g, o.perm, 0, f)
print("rmat 12 ok, max degree", int((g.ptr[1:] - g.ptr[:-1]).max()))

f2 = P.factor_gpu(g, o, 0, P.GpuOptions(watchdog_seconds=1200.0, grid_ctas=2), ctx=ctx)
check(g, o.perm, 0, f2)
print("rmat owner-alone ok")
