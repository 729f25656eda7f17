"""Named inputs shared by the parity tests. Every graph/ordering is built by the
product's host builders (paper_2505_02977_b200), which tests/test_host.py pins
to the reference's generators via tests/golden/golden.json; the names match
golden.json entries produced by tests/golden/make_golden.py."""
import hashlib

import numpy as np

import paper_2505_02977_b200 as P


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def edges_graph(n, edges):
    return P.LaplacianGraph.from_edges(n, edges)


def star(leaves):
    return edges_graph(leaves + 1, [(0, v, 1.0) for v in range(1, leaves + 1)])


def ring(n):
    e = [(v, v + 1, 1.0) for v in range(n - 1)]
    if n > 2:
        e.append((0, n - 1, 1.0))
    return edges_graph(n, e)


def case(name):
    """(graph, perm, seed) for a golden.json factor entry name."""
    I = lambda n: np.arange(n, dtype=np.int32)  # noqa: E731
    if name == "p3":
        return edges_graph(3, [(0, 1, 1.0), (1, 2, 1.0)]), I(3), 0
    if name.startswith("k3_s"):
        return edges_graph(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)]), I(3), int(name[4:])
    if name.startswith("star"):
        k = int(name[4:])
        return star(k), I(k + 1), 0
    if name.startswith("ring"):
        n, s = name[4:].split("_s")
        n, s = int(n), int(s)
        return ring(n), P.ordering_random(n, s).perm, s
    if name.startswith("rc200_s"):
        seed = int(name[7])
        g = P.gen_random_connected(200, 400, seed * 31 + 1)
        if name.endswith("random"):
            return g, P.ordering_random(200, seed).perm, seed
        return g, P.ordering_nnz_sort(g, seed).perm, seed + 1
    if name.startswith("rc50_s"):
        s = int(name[6:])
        return P.gen_random_connected(50, 80, s), P.ordering_random(50, s).perm, s
    if name == "components120":
        return P.gen_random_components(120, 4, 60, 5), P.ordering_random(120, 9).perm, 2
    if name.startswith("components3000_s"):
        s = int(name[16:])
        return P.gen_random_components(3000, 3, 9000, s), P.ordering_random(3000, s).perm, s
    if name.startswith("poisson") and ("_random" in name or "_nnz" in name):
        n = int(name[7:name.index("_")])
        g = P.gen_poisson3d(n)
        tail = name[name.index("_") + 1:]
        if tail.startswith("random"):
            s = int(tail[6:])
            return g, P.ordering_random(n ** 3, s).perm, s
        return g, P.ordering_nnz_sort(g, 0).perm, 0
    if name == "poisson12_contrast":
        g = P.gen_poisson3d(12, "contrast", contrast_ratio=1e4, seed=3)
        return g, P.ordering_random(12 ** 3, 0).perm, 0
    if name == "poisson12_aniso":
        g = P.gen_poisson3d(12, "anisotropic", epsilon=1e-3)
        return g, P.ordering_nnz_sort(g, 0).perm, 0
    raise KeyError(name)


def factor_from_port(f):
    return P.LdlFactor(f["n"], f["col_ptr"], f["rows"], f["values"], f["diag"], f["perm"])
