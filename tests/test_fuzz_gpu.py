"""GPU: seeded structural fuzz of the factorization against the plain-C oracle
(byte-identical factors, proj/tests/test_factor_par.cpp:172-190 style), over
shapes the fixed corpus does not hold: mixed cliques, stars whose hub column
crosses the wide-column threshold (R > 1024), chains, many components, and
weights spread over twelve decades; each case also varies the CTA count."""
import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import factor_from_port

pytestmark = pytest.mark.gpu


def random_graph(rng):
    n = int(rng.integers(2, 3000))
    edges = {}

    def add(u, v):
        if u != v:
            a, b = (u, v) if u < v else (v, u)
            edges[(a, b)] = float(10.0 ** rng.uniform(-6, 6)) if rng.random() < 0.5 else float(rng.integers(1, 5))

    kind = rng.integers(0, 5)
    if kind == 0:  # sparse random
        for _ in range(int(rng.integers(n, 4 * n))):
            add(int(rng.integers(n)), int(rng.integers(n)))
    elif kind == 1:  # a few cliques joined by a chain
        for c in range(int(rng.integers(1, 4))):
            vs = rng.choice(n, size=min(n, int(rng.integers(2, 70))), replace=False)
            for i in range(len(vs)):
                for j in range(i + 1, len(vs)):
                    add(int(vs[i]), int(vs[j]))
        for v in range(n - 1):
            add(v, v + 1)
    elif kind == 2:  # hubs (wide columns) over a ring
        n = int(rng.integers(3000, 6000))
        for v in range(n):
            add(v, (v + 1) % n)
        for h in rng.choice(n, size=int(rng.integers(1, 4)), replace=False):
            for v in rng.choice(n, size=int(rng.integers(1000, n)), replace=False):
                add(int(h), int(v))
    elif kind == 3:  # many small components and isolated vertices
        for _ in range(int(rng.integers(0, 2 * n))):
            u = int(rng.integers(n))
            add(u, min(n - 1, u + int(rng.integers(1, 4))))
    else:  # grid with random extra long-range edges
        s = max(2, int(np.sqrt(n)))
        n = s * s
        for i in range(s):
            for j in range(s):
                if i + 1 < s:
                    add(i * s + j, (i + 1) * s + j)
                if j + 1 < s:
                    add(i * s + j, i * s + j + 1)
        for _ in range(int(rng.integers(0, n // 4 + 1))):
            add(int(rng.integers(n)), int(rng.integers(n)))
    return P.LaplacianGraph.from_edges(n, [(a, b, w) for (a, b), w in edges.items()]), int(kind)


@pytest.mark.parametrize("case_seed", range(64))
def test_fuzz_byte_identical(gpu_ctx, port, case_seed):
    rng = np.random.default_rng(1000 + case_seed)
    g, kind = random_graph(rng)
    seed = int(rng.integers(0, 1 << 31))
    perm = P.ordering_random(g.n, seed).perm if rng.random() < 0.7 else P.ordering_nnz_sort(g, seed).perm
    opts = dict(grid_ctas=int(rng.choice([0, 1, 7, 300])), verify=True)  # 0: the default grid
    st = P.FactorStats()
    f = P.factor_gpu(g, P.Ordering(perm), seed, P.GpuOptions(**opts), st, ctx=gpu_ctx)
    want = port.factor(g, perm, seed)
    assert f.same_values(factor_from_port(want)), (case_seed, kind, g.n)
    assert np.array_equal(st.fills_received, want["fills_received"]), (case_seed, kind)


@pytest.mark.parametrize("case_seed", range(24))
def test_fuzz_solve(gpu_ctx, port, case_seed):
    # apply_preconditioner: exact sweeps bit-identical to the oracle
    # (proj/src/solver.cpp apply_preconditioner), fast sweeps within 1e-10;
    # PCG iterations within 10% of the oracle's
    rng = np.random.default_rng(5000 + case_seed)
    g, kind = random_graph(rng)
    seed = int(rng.integers(0, 1 << 31))
    perm = P.ordering_random(g.n, seed).perm
    want = port.factor(g, perm, seed)
    f = factor_from_port(want)
    r = P.make_rhs(g, "random_projected", seed)
    zref = port.apply_preconditioner(want, r)
    try:
        gpu_ctx.set_preconditioner_mode("exact")
        assert P.apply_preconditioner_gpu(f, r, ctx=gpu_ctx).tobytes() == zref.tobytes(), (case_seed, kind)
        gpu_ctx.set_preconditioner_mode("fast")
        z = P.apply_preconditioner_gpu(f, r, ctx=gpu_ctx)
        assert np.allclose(z, zref, rtol=1e-10, atol=1e-12 * max(np.abs(zref).max(), 1e-300)), (case_seed, kind)
    finally:
        gpu_ctx.set_preconditioner_mode("default")
    rc, _, ref = port.pcg(g, want, r, tol=1e-8)
    try:
        x, rep = P.pcg_solve_gpu(g, f, r, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    except P.Error:
        assert rc != 0 or not ref["converged"], (case_seed, kind)
        return
    # the iteration gate applies where the reference converges (disconnected graphs and
    # twelve-decade weights can stall both; there only a clean report is required)
    if rc == 0 and ref["converged"]:
        assert rep.converged and rep.relative_residual <= 1e-8, (case_seed, kind)
        assert abs(rep.iterations - ref["iterations"]) <= max(1, ref["iterations"] // 10), (case_seed, kind, ref)
    assert np.isfinite(x).all() and rep.iterations <= 1000


@pytest.mark.parametrize("batch_seed", range(6))
def test_fuzz_batch(gpu_ctx, port, batch_seed):
    # config[4]: a batch of random graphs (1-12 of them, hubs included) in one
    # device pass; every member byte-identical to its stand-alone oracle factor
    rng = np.random.default_rng(9000 + batch_seed)
    graphs, perms, seeds = [], [], []
    for _ in range(int(rng.integers(1, 13))):
        g, _ = random_graph(rng)
        s = int(rng.integers(0, 1 << 31))
        graphs.append(g)
        seeds.append(s)
        perms.append(P.ordering_random(g.n, s).perm)
    fs, _ = P.factor_batch_gpu(graphs, [P.Ordering(p) for p in perms], seeds, ctx=gpu_ctx)
    for i, (g, p, s, f) in enumerate(zip(graphs, perms, seeds, fs)):
        assert f.same_values(factor_from_port(port.factor(g, p, s))), (batch_seed, i, g.n)
