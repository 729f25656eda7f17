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
