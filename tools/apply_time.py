import sys, time
sys.path.insert(0, '/root/repo')
import paper_2505_02977_b200 as P
g = P.gen_poisson3d(128); o = P.ordering_random(g.n, 0)
ctx = P.GpuContext(0)
f = P.factor_gpu(g, o, 0, ctx=ctx)
b = P.make_rhs(g, "random_projected", 0)
for mode in ("exact", "fast"):
    ctx.set_preconditioner_mode(mode)
    P.apply_preconditioner_gpu(f, b, ctx=ctx)
    t = time.perf_counter()
    for _ in range(5): P.apply_preconditioner_gpu(f, b, ctx=ctx)
    print(mode, (time.perf_counter() - t) / 5 * 1e3, "ms per apply (wall, incl. H2D/D2H of 16 MB)")
