"""CPU: the C-ABI library loads, exports every symbol include/parac_gpu.h
declares, and its host builders (graphs, orderings, rhs) equal the reference's."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import digest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "parac_gpu.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(parac_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(P.LIB_PATH)
    syms = declared_symbols()
    assert len(syms) >= 30
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2505_02977_b200 import _lib
    assert set(_lib.SIGNATURES) == set(syms)


def test_errc_names_match_reference():
    # proj/src/error.cpp:5-27
    lib = P.rchol.lib
    assert lib.parac_errc_name(10) == b"ArenaExhausted"
    assert lib.parac_errc_name(11) == b"QueueStall"
    assert lib.parac_errc_name(14) == b"NotConnected"
    assert [e.value for e in P.Errc][0] == 1 and P.Errc.internal_error == 17


def build_named(name):
    if name == "poisson16":
        return P.gen_poisson3d(16)
    if name == "poisson12_contrast":
        return P.gen_poisson3d(12, "contrast", contrast_ratio=1e4, seed=3)
    if name == "poisson12_aniso":
        return P.gen_poisson3d(12, "anisotropic", epsilon=1e-3)
    if name == "rc200_1":
        return P.gen_random_connected(200, 400, 1)
    if name == "components120":
        return P.gen_random_components(120, 4, 60, 5)
    raise KeyError(name)


def test_generators_equal_reference(gold):
    for e in gold["graphs"]:
        g = build_named(e["name"])
        assert g.n == e["n"]
        assert digest(g.ptr, g.adj, g.w, g.wdeg) == e["digest"], e["name"]


def test_orderings_equal_reference(gold):
    for e in gold["orderings"]:
        if e["kind"] == "random":
            perm = P.ordering_random(e["n"], e["seed"]).perm
        else:
            perm = P.ordering_nnz_sort(build_named(e["graph"]), e["seed"]).perm
        assert digest(perm) == e["digest"]


def test_from_edges_validation():
    # LaplacianGraph::from_edges rejects these (src/graph.cpp:25-39, :61-66)
    for edges in ([(0, 0, 1.0)], [(0, 1, 0.0)], [(0, 1, -1.0)], [(0, 1, 1.0), (1, 0, 2.0)],
                  [(0, 5, 1.0)]):
        with pytest.raises(P.Error) as ei:
            P.LaplacianGraph.from_edges(3, edges)
        assert ei.value.code == P.Errc.internal_error


def test_ordering_validation():
    with pytest.raises(P.Error) as ei:
        P.Ordering(np.array([0, 0, 1], np.int32))
    assert ei.value.code == P.Errc.not_a_permutation
    with pytest.raises(P.Error):
        P.Ordering(np.array([0, 3, 1], np.int32))


def test_make_rhs_matches_oracle(port):
    for g in (P.gen_poisson3d(8), P.gen_random_connected(100, 200, 3)):
        for mode, name in ((1, "random_projected"), (2, "from_random_x")):
            assert P.make_rhs(g, name, 5).tobytes() == port.make_rhs(g, mode, 5).tobytes()


def test_paper_configs_build():
    g2 = P.gen_poisson2d(16)
    assert g2.n == 256 and g2.num_edges() == 2 * 16 * 15
    g27 = P.gen_poisson27(6)
    # 3 axis + 6 face-diagonal + 4 body-diagonal directions
    assert g27.num_edges() == 3 * 5 * 36 + 6 * 25 * 6 + 4 * 125
    assert (g27.w >= 0.5).all() and (g27.w < 2.0).all()
    gr = P.gen_rmat(10, 8, 0)
    assert gr.n == 1024 and gr.num_edges() > 4000
    assert (gr.adj != np.repeat(np.arange(gr.n), np.diff(gr.ptr))).all()


def test_no_cpu_fallback_without_device():
    if P.device_count() > 0:
        pytest.skip("a CUDA device is present")
    with pytest.raises(P.Error) as ei:
        P.GpuContext(0)
    assert "no CPU fallback" in str(ei.value)
