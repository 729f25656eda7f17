"""GPU: the solve path. laplacian_apply and apply_preconditioner are
bit-identical to the reference order (proj/src/solver.cpp:32-93); PCG reaches
the tolerance with an iteration count within 10% of the reference's
(BASELINE north_star), with the reference's error behaviour."""
import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import case, digest, factor_from_port

pytestmark = pytest.mark.gpu


def test_laplacian_apply_bit_exact(gpu_ctx, port):
    for g in (P.gen_poisson3d(10), P.gen_random_connected(500, 2000, 2), P.gen_poisson27(6)):
        x = P.make_rhs(g, "random_projected", 3)
        assert P.laplacian_apply_gpu(g, x, ctx=gpu_ctx).tobytes() == port.laplacian_apply(g, x).tobytes()


def test_preconditioner_p3_by_hand(gpu_ctx, port):
    # proj/tests/test_solver.cpp:27-35: exact P3 factor, r = (1,0,-1) -> z = (2,1,0)
    g, perm, _ = case("p3")
    f = factor_from_port(port.factor(g, perm, 0, exact=True))
    z = P.apply_preconditioner_gpu(f, np.array([1.0, 0.0, -1.0]), ctx=gpu_ctx)
    assert z.tolist() == [2.0, 1.0, 0.0]
    assert P.apply_preconditioner_gpu(f, np.zeros(3), ctx=gpu_ctx).tolist() == [0.0, 0.0, 0.0]
    empty = P.LaplacianGraph.from_edges(3, [])
    fe = P.factor_gpu(empty, P.Ordering.identity(3), 0, ctx=gpu_ctx)
    assert P.apply_preconditioner_gpu(fe, np.array([3.0, -1.0, 5.0]), ctx=gpu_ctx).tolist() == [0.0] * 3
    with pytest.raises(P.Error) as ei:
        P.apply_preconditioner_gpu(f, np.ones(2), ctx=gpu_ctx)
    assert ei.value.code == P.Errc.dimension_mismatch


def test_preconditioner_bit_exact(gpu_ctx, port, gold):
    e = gold["precond"][0]
    g = P.gen_random_connected(300, 700, 4)
    f = port.factor(g, P.ordering_random(300, 2).perm, e["seed"])
    r = P.make_rhs(g, "random_projected", e["rhs_seed"])
    z = P.apply_preconditioner_gpu(factor_from_port(f), r, ctx=gpu_ctx)
    assert digest(z) == e["z_digest"]
    for name in ("poisson16_random0", "poisson32_nnz0", "components3000_s1"):
        g, perm, seed = case(name)
        f = port.factor(g, perm, seed)
        r = P.make_rhs(g, "random_projected", 1)
        z = P.apply_preconditioner_gpu(factor_from_port(f), r, ctx=gpu_ctx)
        assert z.tobytes() == port.apply_preconditioner(f, r).tobytes(), name


def test_schedule_levels_match(gpu_ctx, port, gold):
    for name in ("p3", "poisson16_random0", "rc200_s0_nnz", "components3000_s2"):
        g, perm, seed = case(name)
        f = port.factor(g, perm, seed)
        lv, depth = P.schedule_levels_gpu(factor_from_port(f), ctx=gpu_ctx)
        want_lv, want_depth = port.schedule_levels(f)
        assert depth == want_depth and np.array_equal(lv, want_lv), name


def test_pcg_iterations_within_10pct(gpu_ctx, gold):
    for e in gold["pcg"]:
        name = e["name"]
        n = int(name[7:name.index("_")])
        g = P.gen_poisson3d(n)
        o = P.ordering_nnz_sort(g, 0) if "_nnz" in name else P.ordering_random(n ** 3, 0)
        f = P.factor_gpu(g, o, e["seed"], ctx=gpu_ctx)
        b = P.make_rhs(g, "random_projected", e["rhs_seed"])
        x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=e["tol"]), ctx=gpu_ctx)
        assert rep.converged and rep.relative_residual <= e["tol"]
        assert abs(rep.iterations - e["iterations"]) <= max(1, 0.1 * e["iterations"]), (name, rep.iterations)
        assert rep.recurrence_residual == pytest.approx(rep.relative_residual, rel=1e-3)
        assert abs(x.mean()) < 1e-12


def test_pcg_exact_factor_immediate(gpu_ctx, port):
    # proj/tests/test_solver.cpp:77-113
    for seed in range(4):
        n = 20 + 30 * (seed % 4)
        g = P.gen_random_connected(n, 2 * n, seed)
        f = factor_from_port(port.factor(g, P.ordering_random(n, seed).perm, 0, exact=True))
        b = P.make_rhs(g, "from_random_x", seed)
        x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(), ctx=gpu_ctx)
        assert rep.converged and rep.iterations <= 3 and rep.relative_residual <= 1e-10


def test_pcg_errors_and_limits(gpu_ctx):
    # proj/tests/test_solver.cpp:128-150
    g = P.gen_random_components(20, 2, 10, 3)
    f = P.factor_gpu(g, P.Ordering.identity(20), 0, ctx=gpu_ctx)
    b = np.zeros(20)
    b[0], b[1] = 1.0, -1.0
    with pytest.raises(P.Error) as ei:
        P.pcg_solve_gpu(g, f, b, ctx=gpu_ctx)
    assert ei.value.code == P.Errc.not_connected
    g = P.gen_poisson3d(8)
    f = P.factor_gpu(g, P.ordering_random(512, 0), 0, ctx=gpu_ctx)
    b = P.make_rhs(g, "random_projected", 2)
    x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-14, max_iters=3), ctx=gpu_ctx)
    assert rep.iterations == 3 and not rep.converged
    x, rep = P.pcg_solve_gpu(g, f, np.zeros(512), ctx=gpu_ctx)
    assert rep.converged and rep.iterations == 0 and not x.any()


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_pcg_modes_iterations(gpu_ctx, gold, mode):
    # both sweep modes: same operator M^-1; iterations within 10% of the reference
    e = next(x for x in gold["pcg"] if x["name"] == "poisson32_random_1e-8")
    g = P.gen_poisson3d(32)
    f = P.factor_gpu(g, P.ordering_random(32 ** 3, 0), e["seed"], ctx=gpu_ctx)
    b = P.make_rhs(g, "random_projected", e["rhs_seed"])
    gpu_ctx.set_preconditioner_mode(mode)
    try:
        x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
        x2, rep2 = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    finally:
        gpu_ctx.set_preconditioner_mode("default")
    assert rep.converged and rep.relative_residual <= 1e-8
    assert abs(rep.iterations - e["iterations"]) <= max(1, 0.1 * e["iterations"])
    assert x.tobytes() == x2.tobytes()  # deterministic run to run


def test_fast_preconditioner_close_to_exact(gpu_ctx, port):
    g, perm, seed = case("poisson16_random0")
    f = port.factor(g, perm, seed)
    r = P.make_rhs(g, "random_projected", 3)
    want = port.apply_preconditioner(f, r)
    gpu_ctx.set_preconditioner_mode("fast")
    try:
        z = P.apply_preconditioner_gpu(factor_from_port(f), r, ctx=gpu_ctx)
    finally:
        gpu_ctx.set_preconditioner_mode("default")
    assert np.allclose(z, want, rtol=1e-10, atol=1e-12 * np.abs(want).max())


def test_resident_factor_tracking_across_batch(gpu_ctx):
    # factor_gpu keeps its factor resident; a batch pass replaces the device
    # state, and later solves on the single factor must re-stage it
    g = P.gen_poisson3d(10)
    o = P.ordering_random(g.n, 2)
    f = P.factor_gpu(g, o, 2, ctx=gpu_ctx)
    b = P.make_rhs(g, "random_projected", 0)
    z0 = P.apply_preconditioner_gpu(f, b, ctx=gpu_ctx)
    P.factor_batch_gpu([P.gen_poisson3d(6), P.gen_poisson3d(7)], [P.ordering_random(216, 0),
                       P.ordering_random(343, 1)], [0, 1], ctx=gpu_ctx)
    z1 = P.apply_preconditioner_gpu(f, b, ctx=gpu_ctx)
    assert z0.tobytes() == z1.tobytes()
    x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    assert rep.converged
    assert not f.values.flags.writeable  # factors from factor_gpu are immutable


def test_fast_pcg_deterministic_across_builds(gpu_ctx):
    # the fast PCG's summation orders follow the level-order layout, which is
    # a stable sort of the factor: every build of the same factor (a re-upload,
    # another context) gives the same bits, graph-driven or not
    g = P.gen_poisson3d(30)  # n = 27000: above the exact threshold
    o = P.ordering_random(g.n, 5)
    f = P.factor_gpu(g, o, 5, ctx=gpu_ctx)
    b = P.make_rhs(g, "random_projected", 2)
    x1, r1 = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    x2, r2 = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)  # graph replay
    f2 = P.LdlFactor(f.n, f.col_ptr, f.rows, f.values, f.diag, f.perm)  # same arrays, new object: re-upload
    x3, r3 = P.pcg_solve_gpu(g, f2, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    with P.GpuContext(0) as other:
        x4, r4 = P.pcg_solve_gpu(g, f2, b, P.SolveConfig(tol=1e-8), ctx=other)
    assert not r1.exact and r1.converged
    for x, r in ((x2, r2), (x3, r3), (x4, r4)):
        assert x.tobytes() == x1.tobytes() and r.iterations == r1.iterations
        assert r.relative_residual == r1.relative_residual
