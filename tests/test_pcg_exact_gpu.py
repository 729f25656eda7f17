"""GPU: the exact PCG is pcg_solve (proj/src/solver.cpp:95-175) bit for bit --
x, the iteration count, both residuals and the converged flag are the
reference's bytes. parac_gpu_pcg runs it by default for n <= 16384 and on
request (mode "exact") at any size; above that the fast PCG keeps the
north_star's statistical gate (iterations within 10%).

The FLAG seeds are the round-1 fuzz cases (profiles/fuzz_r01/
fuzz_solve_0_1500.log) whose ill-conditioned hub graphs put the fast PCG's
true residual just above tol (converged = false) where the reference's landed
just below: with the exact PCG the flag is the reference's own."""
import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import digest, factor_from_port
from test_fuzz_gpu import random_graph

pytestmark = pytest.mark.gpu

FLAG_SEEDS = [523, 631, 841, 965, 1047, 1095, 1319, 1410]


def _solve_case(cs):
    rng = np.random.default_rng(5000 + cs)
    g, kind = random_graph(rng)
    seed = int(rng.integers(0, 1 << 31))
    return g, kind, seed


def _same_report(rep, ref):
    return (rep.iterations == ref["iterations"] and rep.converged == ref["converged"]
            and rep.relative_residual == ref["relative_residual"]
            and rep.recurrence_residual == ref["recurrence_residual"])


@pytest.mark.parametrize("cs", FLAG_SEEDS)
def test_flag_seeds_converged_equals_reference(gpu_ctx, port, cs):
    g, kind, seed = _solve_case(cs)
    want = port.factor(g, P.ordering_random(g.n, seed).perm, seed)
    f = factor_from_port(want)
    r = P.make_rhs(g, "random_projected", seed)
    rc, xref, ref = port.pcg(g, want, r, tol=1e-8)
    assert rc == 0 and ref["converged"]  # the reference converges on every FLAG seed
    x, rep = P.pcg_solve_gpu(g, f, r, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)  # default mode
    assert rep.exact, "n <= 16384 must take the exact PCG by default"
    assert rep.converged == ref["converged"] and rep.relative_residual <= 1e-8, (cs, kind)
    assert _same_report(rep, ref), (cs, rep, ref)
    assert x.tobytes() == xref.tobytes()


@pytest.mark.parametrize("case_seed", range(0, 48, 2))
def test_exact_pcg_bytes_fuzz(gpu_ctx, port, case_seed):
    g, kind, seed = _solve_case(case_seed)
    want = port.factor(g, P.ordering_random(g.n, seed).perm, seed)
    f = factor_from_port(want)
    r = P.make_rhs(g, "random_projected", seed)
    rc, xref, ref = port.pcg(g, want, r, tol=1e-8)
    try:
        x, rep = P.pcg_solve_gpu(g, f, r, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    except P.Error as e:
        assert rc != 0 and e.code == rc  # not_connected, like the reference
        return
    assert rc == 0 and rep.exact
    assert _same_report(rep, ref), (case_seed, kind, rep, ref)
    assert x.tobytes() == xref.tobytes()


def test_exact_pcg_golden_digests(gpu_ctx, gold):
    # reference-generated digests of x (tests/golden/make_golden.py), in exact
    # mode at every size, including 32^3 (n = 32768 > the default threshold)
    gpu_ctx.set_preconditioner_mode("exact")
    try:
        for e in gold["pcg"]:
            name = e["name"]
            n = int(name[7:name.index("_")])
            g = P.gen_poisson3d(n)
            o = P.ordering_nnz_sort(g, 0) if "_nnz" in name else P.ordering_random(n ** 3, 0)
            f = P.factor_gpu(g, o, e["seed"], ctx=gpu_ctx)
            b = P.make_rhs(g, "random_projected", e["rhs_seed"])
            x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=e["tol"]), ctx=gpu_ctx)
            assert rep.exact
            assert rep.iterations == e["iterations"], name
            assert rep.relative_residual == e["relative_residual"], name
            assert rep.recurrence_residual == e["recurrence_residual"], name
            assert digest(x) == e["x_digest"], name
    finally:
        gpu_ctx.set_preconditioner_mode("default")


def test_default_mode_switches_to_fast_above_threshold(gpu_ctx, port):
    g = P.gen_poisson3d(26)  # n = 17576 > 16384
    o = P.ordering_random(g.n, 0)
    f = P.factor_gpu(g, o, 0, ctx=gpu_ctx)
    b = P.make_rhs(g, "random_projected", 0)
    x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    rc, _, ref = port.pcg(g, port.factor(g, o.perm, 0), b, tol=1e-8)
    assert not rep.exact and rep.converged
    assert abs(rep.iterations - ref["iterations"]) <= max(1, ref["iterations"] // 10)


def test_exact_pcg_edge_cases(gpu_ctx, port):
    # zero right-hand side (solver.cpp:110-115), max_iters cap, a single edge
    g = P.gen_poisson3d(6)
    o = P.ordering_random(g.n, 3)
    want = port.factor(g, o.perm, 3)
    f = factor_from_port(want)
    x, rep = P.pcg_solve_gpu(g, f, np.zeros(g.n), ctx=gpu_ctx)
    assert rep.exact and rep.converged and rep.iterations == 0 and not x.any()
    b = P.make_rhs(g, "random_projected", 1)
    x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-14, max_iters=2), ctx=gpu_ctx)
    rc, xref, ref = port.pcg(g, want, b, tol=1e-14, max_iters=2)
    assert _same_report(rep, ref) and x.tobytes() == xref.tobytes() and rep.iterations == 2
    g2 = P.LaplacianGraph.from_edges(2, [(0, 1, 2.5)])
    o2 = P.Ordering.identity(2)
    w2 = port.factor(g2, o2.perm, 0)
    b2 = np.array([1.0, -1.0])
    x, rep = P.pcg_solve_gpu(g2, factor_from_port(w2), b2, ctx=gpu_ctx)
    rc, xref, ref = port.pcg(g2, w2, b2, tol=1e-6)
    assert _same_report(rep, ref) and x.tobytes() == xref.tobytes()
