"""PCG and the exact preconditioner on a hub graph (largest connected component
of R-MAT 14): G's transposed rows reach thousands of entries, which takes the
long-row transpose path (CUB segmented sort) of the solve setup. The exact
preconditioner must stay bit-identical to the reference's apply_preconditioner
(solver.cpp:32-74), and PCG must converge within 10% of the reference's
iterations (north_star)."""
import numpy as np
import pytest

import oracle
import paper_2505_02977_b200 as P

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.Reference.available(), reason="oracle/_ref not built")]


def largest_component(g, R):
    h = R.graph_from_csr(g)
    lab = np.empty(g.n, np.int32)
    cnt = oracle.C.c_int32()
    R._chk(R.L.pref_connected_components(h, lab.ctypes.data, oracle.C.byref(cnt)))
    R.free_graph(h)
    big = np.bincount(lab).argmax()
    keep = np.flatnonzero(lab == big)
    remap = -np.ones(g.n, np.int64)
    remap[keep] = np.arange(len(keep))
    src = np.repeat(np.arange(g.n), np.diff(g.ptr))
    m = (lab[src] == big) & (g.adj > src)
    return P.LaplacianGraph.from_edges(len(keep), list(zip(remap[src[m]].tolist(), remap[g.adj[m]].tolist(),
                                                              g.w[m].tolist())))


def test_hub_graph_pcg_and_exact_preconditioner(gpu_ctx):
    R = oracle.Reference()
    g = largest_component(P.gen_rmat(14, 16, 0), R)
    o = P.ordering_random(g.n, 0)
    f = P.factor_gpu(g, o, 0, ctx=gpu_ctx)
    assert np.bincount(f.rows, minlength=g.n).max() > 256  # long transposed rows exist
    b = P.make_rhs(g, "random_projected", 0)
    h = R.graph_from_csr(g)
    fr, _ = R.factor(h, o.perm, 0, backend=R.SEQ)
    z = P.apply_preconditioner_gpu(f, b, ctx=gpu_ctx)
    zr = np.empty(g.n)
    R._chk(R.L.pref_apply_preconditioner(fr, b.ctypes.data, zr.ctypes.data))
    assert z.tobytes() == zr.tobytes()
    x, rep = P.pcg_solve_gpu(g, f, b, P.SolveConfig(tol=1e-8), ctx=gpu_ctx)
    it, conv = oracle.C.c_int(), oracle.C.c_int()
    rel, rec, sec = oracle.C.c_double(), oracle.C.c_double(), oracle.C.c_double()
    xr = np.empty(g.n)
    R._chk(R.L.pref_pcg(h, fr, b.ctypes.data, 1e-8, 1000, xr.ctypes.data, oracle.C.byref(it), oracle.C.byref(rel),
                        oracle.C.byref(rec), oracle.C.byref(conv), oracle.C.byref(sec)))
    assert rep.converged and rep.relative_residual <= 1e-8
    assert abs(rep.iterations - it.value) <= max(1, it.value // 10), (rep.iterations, it.value)
    R.free_factor(fr)
    R.free_graph(h)
