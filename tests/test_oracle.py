"""CPU: pin the C restatement (oracle/rchol_oracle.c) to the reference.

Sources of truth: the reference's own known-answer tests (proj/tests/*.cpp,
cited per test) and tests/golden/golden.json, produced by the unmodified
reference build (tests/golden/make_golden.py)."""
import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import case, digest


def test_unit_uniform_matches_reference_stream(port, ref):
    for seed, key, ctr in [(0, 0, 0), (1, 5, 7), (2**63 + 11, -3, 12345), (42, 2**40, 2**33)]:
        assert port.unit_uniform(seed, key, ctr) == ref.L.pref_unit_uniform(seed, key, ctr)
        assert port.derive_seed(seed, 0x73616D706C696E67) == ref.L.pref_derive_seed(seed, 0x73616D706C696E67)


def test_p3_by_hand(port):
    # proj/tests/test_factor_seq.cpp:14-24
    g, perm, seed = case("p3")
    f = port.factor(g, perm, seed)
    assert f["col_ptr"].tolist() == [0, 1, 2, 2]
    assert f["rows"].tolist() == [1, 2]
    assert f["values"].tolist() == [-1.0, -1.0]
    assert f["diag"].tolist() == [1.0, 1.0, 0.0]
    assert port.factor(g, perm, 0, exact=True)["values"].tolist() == [-1.0, -1.0]


@pytest.mark.parametrize("seed", [0, 7, 123456])
def test_k3_deterministic(port, seed):
    # proj/tests/test_factor_seq.cpp:26-34
    g, perm, _ = case("k3_s0")
    f = port.factor(g, perm, seed)
    assert f["values"].tolist() == [-0.5, -0.5, -1.0]
    assert f["diag"].tolist() == [2.0, 1.5, 0.0]


def test_single_vertex(port):
    # proj/tests/test_factor_seq.cpp:36-41
    g = P.LaplacianGraph.from_edges(1, [])
    f = port.factor(g, np.zeros(1, np.int32), 0)
    assert len(f["rows"]) == 0 and f["diag"].tolist() == [0.0]


def test_dependency_counts():
    # proj/tests/test_factor_seq.cpp:43-54
    from corpus import star
    assert P.dependency_counts(star(3), P.Ordering.identity(4)).tolist() == [0, 1, 1, 1]
    g, _, _ = case("p3")
    assert P.dependency_counts(g, P.Ordering.identity(3)).tolist() == [0, 1, 1]
    for seed in range(5):
        g = P.gen_random_connected(20, 30, seed)
        assert P.dependency_counts(g, P.ordering_random(20, seed))[0] == 0


def test_rings_randomized_equals_exact(port):
    # proj/tests/test_factor_seq.cpp:56-68
    from corpus import ring
    for n in (2, 5, 9):
        for seed in range(4):
            g = ring(n)
            perm = P.ordering_random(n, seed).perm
            a, b = port.factor(g, perm, seed), port.factor(g, perm, seed, exact=True)
            for k in ("col_ptr", "rows", "values", "diag"):
                assert a[k].tobytes() == b[k].tobytes()


def test_fill_accounting(port):
    # proj/tests/test_factor_seq.cpp:70-95
    for seed in range(6):
        g = P.gen_random_connected(50, 80, seed)
        o = P.ordering_random(50, seed)
        f = port.factor(g, o.perm, seed)
        m = f["merged_degree"]
        assert np.array_equal(f["samples_emitted"], np.maximum(m - 1, 0))
        assert f["fills_received"].sum() == f["total_fills"]
        assert m.sum() == len(f["rows"])
        for k in range(50):
            assert m[k] <= g.degree(o.inverse[k]) + f["fills_received"][k]


def test_signs(port):
    # proj/tests/test_factor_seq.cpp:97-104
    for seed in range(6):
        g = P.gen_random_components(80, 1 + seed % 3, 100, seed)
        f = port.factor(g, P.ordering_random(80, seed).perm, seed)
        assert (f["values"] <= 0).all() and (f["diag"] >= 0).all()


def test_star_center_first_rows(port, ref):
    # proj/tests/test_factor_par.cpp:67-103: pick a seed whose first draw pairs
    # leaves 1 and 2; the factor is then a full chain with rows {1,2,3,2,3}.
    from corpus import star
    chosen = next(s for s in range(64)
                  if port.unit_uniform(port.derive_seed(s, 0x73616D706C696E67), 0, 0) * 2.0 >= 1.0)
    f = port.factor(star(3), np.arange(4, dtype=np.int32), chosen)
    assert f["rows"].tolist() == [1, 2, 3, 2, 3]
    # reference dp trace through TestHooks::on_phase: (0,1,2,2) then (0,0,1,1)
    h = ref.graph_from_csr(star(3))
    snaps = np.zeros((4, 4), np.int64)
    cnt = ref_count = __import__("ctypes").c_int()
    fh = __import__("oracle").vp()
    ref._chk(ref.L.pref_factor_left_trace(h, np.arange(4, dtype=np.int32).ctypes.data, chosen, 2, 0,
                                          snaps.ctypes.data, 4, __import__("ctypes").byref(cnt),
                                          __import__("ctypes").byref(fh)))
    assert cnt.value >= 2
    assert snaps[0].tolist() == [0, 1, 2, 2] and snaps[1].tolist() == [0, 0, 1, 1]
    del ref_count


def test_port_matches_golden_factors(port, gold):
    for e in gold["factors"]:
        g, perm, seed = case(e["name"])
        assert digest(perm) == e["perm_digest"], e["name"]
        assert seed == e["seed"]
        f = port.factor(g, perm, seed)
        assert f"{port.checksum(f):016x}" == e["checksum"], e["name"]
        assert digest(f["merged_degree"], f["samples_emitted"], f["fills_received"]) == e["stats_digest"]
        assert f["total_fills"] == e["total_fills"]
        assert port.schedule_levels(f)[1] == e["depth"], e["name"]
        if "arrays" in e:
            for k in ("col_ptr", "rows", "values", "diag"):
                assert f[k].tolist() == e["arrays"][k]


def test_port_matches_golden_pcg(port, gold):
    for e in gold["pcg"]:
        name = e["name"]
        n = int(name[7:name.index("_")])
        g = P.gen_poisson3d(n)
        perm = (P.ordering_nnz_sort(g, 0) if "_nnz" in name else P.ordering_random(n ** 3, 0)).perm
        f = port.factor(g, perm, e["seed"])
        b = port.make_rhs(g, 1, e["rhs_seed"])
        assert digest(b) == e["rhs_digest"]
        rc, x, rep = port.pcg(g, f, b, e["tol"], 1000)
        assert rc == 0
        assert rep["iterations"] == e["iterations"]
        assert rep["relative_residual"] == e["relative_residual"]
        assert digest(x) == e["x_digest"]


def test_port_matches_golden_preconditioner(port, gold):
    e = gold["precond"][0]
    g = P.gen_random_connected(300, 700, 4)
    f = port.factor(g, P.ordering_random(300, 2).perm, e["seed"])
    z = port.apply_preconditioner(f, port.make_rhs(g, 1, e["rhs_seed"]))
    assert digest(z) == e["z_digest"]


def test_port_pcg_rejects_disconnected(port):
    g = P.gen_random_components(20, 2, 10, 3)
    f = port.factor(g, np.arange(20, dtype=np.int32), 0)
    b = np.zeros(20)
    b[0], b[1] = 1.0, -1.0
    assert port.pcg(g, f, b)[0] == 14  # Errc::not_connected


def test_fullsize_fixture_pins_survey_values():
    # tests/golden/fullsize.json (made from oracle/_ref at the BASELINE sizes)
    # agrees with the survey's independent probe.
    import json
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "fullsize.json")) as fh:
        full = {c["name"]: c for c in json.load(fh)["configs"]}
    assert full["poisson3d_128"]["checksum"] == "13308715cf34482c"
    assert full["poisson3d_128"]["nnz_off"] == 22048797
    assert full["poisson3d_128"]["total_fills"] == 19951646
    assert full["poisson3d_128"]["depth"] == 1206
    assert full["poisson3d_128"]["pcg"]["iterations"] == 34
    assert full["poisson2d_256"]["nnz_off"] == 330229 and full["poisson2d_256"]["depth"] == 139
    assert full["poisson2d_256"]["pcg"]["iterations"] == 50
    assert full["rmat_22"]["n"] == 4194304


@pytest.mark.parametrize("kind,size,seed", [("poisson2d", 16, 0), ("poisson27", 6, 1), ("poisson27", 5, 7),
                                            ("rmat", 10, 0), ("rmat", 11, 3)])
def test_harness_generators_match_product(port, ref, kind, size, seed):
    # the reference arm of bench.py builds its inputs from these edge lists and
    # the reference's own from_edges; they must be the product's graphs exactly
    import paper_2505_02977_b200 as P
    g = {"poisson2d": lambda: P.gen_poisson2d(size), "poisson27": lambda: P.gen_poisson27(size, seed),
         "rmat": lambda: P.gen_rmat(size, 16, seed)}[kind]()
    n, a, b, w = port.gen_edges(kind, size, seed)
    h = ref.graph_from_edges(n, a, b, w)
    try:
        rn, ptr, adj, ww, _ = ref.csr(h)
    finally:
        ref.free_graph(h)
    assert rn == g.n and np.array_equal(ptr, g.ptr) and np.array_equal(adj, g.adj)
    assert ww.tobytes() == g.w.tobytes()
