"""Long run of tests/test_fuzz_gpu.py's generator: python tools/fuzz_sweep.py START COUNT [--solve|--batch|--rmat].
Without --solve: factors byte for byte; with it: exact-mode preconditioner bytes,
fast mode within 1e-10, and the default PCG (exact at these sizes) bit-identical
to the oracle's pcg_solve (--fast: the fast PCG, iterations within 10%).
Prints one line per failing case and a summary (GPU; the oracle is the checker)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import oracle  # noqa: E402
import paper_2505_02977_b200 as P  # noqa: E402
from corpus import factor_from_port  # noqa: E402
from test_fuzz_gpu import random_graph  # noqa: E402

start, count = int(sys.argv[1]), int(sys.argv[2])
port, ctx = oracle.Port(), P.GpuContext(0)
bad, t0 = 0, time.time()


def solve_case(cs):
    rng = np.random.default_rng(5000 + cs)
    g, kind = random_graph(rng)
    seed = int(rng.integers(0, 1 << 31))
    want = port.factor(g, P.ordering_random(g.n, seed).perm, seed)
    f = factor_from_port(want)
    r = P.make_rhs(g, "random_projected", seed)
    zref = port.apply_preconditioner(want, r)
    ctx.set_preconditioner_mode("exact")
    if P.apply_preconditioner_gpu(f, r, ctx=ctx).tobytes() != zref.tobytes():
        return f"exact {kind} {g.n}"
    ctx.set_preconditioner_mode("fast")
    z = P.apply_preconditioner_gpu(f, r, ctx=ctx)
    ctx.set_preconditioner_mode("default")
    if not np.allclose(z, zref, rtol=1e-10, atol=1e-12 * max(np.abs(zref).max(), 1e-300)):
        return f"fast {kind} {g.n}"
    rc, xref, ref = port.pcg(g, want, r, tol=1e-8)
    if "--fast" in sys.argv:
        ctx.set_preconditioner_mode("fast")
    try:
        x, rep = P.pcg_solve_gpu(g, f, r, P.SolveConfig(tol=1e-8), ctx=ctx)
    except P.Error as e:
        return None if rc != 0 or not ref["converged"] else f"pcg error {e}"
    finally:
        ctx.set_preconditioner_mode("default")
    what = (f"{kind} {g.n} iters {rep.iterations} vs {ref['iterations']} true/recurrence residual "
            f"{rep.relative_residual:.3g}/{rep.recurrence_residual:.3g} vs "
            f"{ref['relative_residual']:.3g}/{ref['recurrence_residual']:.3g}")
    if rep.exact:
        # default mode at these sizes: the exact PCG, bit-identical to pcg_solve
        same = (rep.iterations == ref["iterations"] and rep.converged == ref["converged"]
                and rep.relative_residual == ref["relative_residual"]
                and rep.recurrence_residual == ref["recurrence_residual"])
        return None if same and x.tobytes() == xref.tobytes() else "exact pcg " + what
    if rc == 0 and ref["converged"]:
        it_ok = abs(rep.iterations - ref["iterations"]) <= max(1, ref["iterations"] // 10)
        if not it_ok:
            return "pcg " + what
        if not rep.converged:
            # both stop on the recurrence residual; the true residual of an
            # ill-conditioned graph can land either side of tol
            print("FLAG", cs, what, flush=True)
    return None


def batch_case(cs):
    rng = np.random.default_rng(9000 + cs)
    graphs, perms, seeds = [], [], []
    for _ in range(int(rng.integers(1, 13))):
        g, _ = random_graph(rng)
        s = int(rng.integers(0, 1 << 31))
        graphs.append(g)
        seeds.append(s)
        perms.append(P.ordering_random(g.n, s).perm)
    fs, _ = P.factor_batch_gpu(graphs, [P.Ordering(p) for p in perms], seeds, ctx=ctx)
    for i, (g, p, s, f) in enumerate(zip(graphs, perms, seeds, fs)):
        if not f.same_values(factor_from_port(port.factor(g, p, s))):
            return f"batch member {i} n={g.n}"
    return None


def rmat_case(cs):
    # R-MAT graphs of scales 10-14 (hub columns: several cooperative jobs at
    # once), random or nnz-sort orderings, grids from 2 CTAs (owner alone) to
    # the full co-resident grid
    rng = np.random.default_rng(7000 + cs)
    scale = 10 + cs % 5
    g = P.gen_rmat(scale, int(rng.integers(8, 24)), int(rng.integers(0, 1 << 30)))
    seed = int(rng.integers(0, 1 << 31))
    o = P.ordering_random(g.n, seed) if cs % 3 else P.ordering_nnz_sort(g, seed)
    grid = int(rng.choice([0, 0, 2, 9, 37]))
    f = P.factor_gpu(g, o, seed, P.GpuOptions(grid_ctas=grid), ctx=ctx)
    if not f.same_values(factor_from_port(port.factor(g, o.perm, seed))):
        return f"rmat scale {scale} grid {grid} n={g.n}"
    return None


if "--rmat" in sys.argv:
    for cs in range(start, start + count):
        msg = rmat_case(cs)
        if msg:
            bad += 1
            print("MISMATCH", cs, msg, flush=True)
    print(f"rmat cases {count} mismatches {bad} seconds {time.time() - t0:.1f}")
    sys.exit(0)
if "--batch" in sys.argv:
    for cs in range(start, start + count):
        msg = batch_case(cs)
        if msg:
            bad += 1
            print("MISMATCH", cs, msg, flush=True)
    print(f"batch cases {count} mismatches {bad} seconds {time.time() - t0:.1f}")
    sys.exit(0)
if "--solve" in sys.argv:
    for cs in range(start, start + count):
        msg = solve_case(cs)
        if msg:
            bad += 1
            print("MISMATCH", cs, msg, flush=True)
    print(f"solve cases {count} mismatches {bad} seconds {time.time() - t0:.1f}")
    sys.exit(0)
for cs in range(start, start + count):
    rng = np.random.default_rng(1000 + cs)
    g, kind = random_graph(rng)
    seed = int(rng.integers(0, 1 << 31))
    perm = P.ordering_random(g.n, seed).perm if rng.random() < 0.7 else P.ordering_nnz_sort(g, seed).perm
    opts = dict(grid_ctas=int(rng.choice([0, 1, 7, 300])), verify=True)
    try:
        f = P.factor_gpu(g, P.Ordering(perm), seed, P.GpuOptions(**opts), ctx=ctx)
        ok = f.same_values(factor_from_port(port.factor(g, perm, seed)))
    except P.Error as e:
        ok = False
        print("error", cs, kind, g.n, e, flush=True)
    if not ok:
        bad += 1
        print("MISMATCH", cs, kind, g.n, opts, flush=True)
print(f"cases {count} mismatches {bad} seconds {time.time() - t0:.1f}")
