"""TEST INFRASTRUCTURE ONLY — the checker, never the product.

Two CPU oracles for the rchol hot path, importable only from tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / reference arm:

  * `port`      : oracle/rchol_oracle.c, a plain-C restatement of the reference
                  (liboracle.so in oracle/_build). Always available once built.
  * `reference` : the UNMODIFIED reference library compiled from
                  /root/reference/proj/src by oracle/Makefile into
                  oracle/_ref/libparac_ref.so, driven through ref_driver.cpp.
                  Built in the dev container; the built .so travels to GPU boxes.

Parity of the port is pinned by tests/test_oracle.py (reference known-answer
tests + golden vectors in tests/golden/ produced by the reference build).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_LIB = os.path.join(HERE, "_build", "liboracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libparac_ref.so")

vp, i32, i64, u64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double


def build(reference: bool = True) -> None:
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)
    if reference and os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", HERE, "ref"], check=True)


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


class OracleFactor(C.Structure):
    _fields_ = [("n", i32), ("col_ptr", C.POINTER(i64)), ("rows", C.POINTER(i32)),
                ("values", C.POINTER(f64)), ("diag", C.POINTER(f64)),
                ("merged_degree", C.POINTER(i32)), ("samples_emitted", C.POINTER(i32)),
                ("fills_received", C.POINTER(i32)), ("total_fills", i64)]


class Port:
    """ctypes view of oracle/rchol_oracle.c."""

    def __init__(self, path: str = PORT_LIB):
        if not os.path.exists(path):
            build(reference=False)
        L = C.CDLL(path)
        L.oracle_unit_uniform.restype = f64
        L.oracle_unit_uniform.argtypes = [u64, i64, u64]
        L.oracle_derive_seed.restype = u64
        L.oracle_derive_seed.argtypes = [u64, u64]
        L.oracle_factor_randomized.argtypes = [i32, vp, vp, vp, vp, u64, C.c_int, C.POINTER(OracleFactor)]
        L.oracle_factor_free.argtypes = [C.POINTER(OracleFactor)]
        L.oracle_checksum.restype = u64
        L.oracle_checksum.argtypes = [i32, vp, vp, vp, vp]
        L.oracle_schedule_levels.restype = i32
        L.oracle_schedule_levels.argtypes = [i32, vp, vp, vp]
        L.oracle_apply_preconditioner.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_laplacian_apply.argtypes = [i32, vp, vp, vp, vp, vp]
        L.oracle_make_rhs.argtypes = [i32, vp, vp, vp, C.c_int, u64, vp]
        L.oracle_pcg.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, f64, C.c_int, vp,
                                 C.POINTER(C.c_int), C.POINTER(f64), C.POINTER(f64), C.POINTER(C.c_int)]
        L.oracle_build_pos_graph.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, vp]
        L.oracle_gen_edges.restype = i64
        L.oracle_gen_edges.argtypes = [C.c_int, i32, u64, C.POINTER(C.POINTER(i32)), C.POINTER(C.POINTER(i32)),
                                       C.POINTER(C.POINTER(f64)), C.POINTER(i32)]
        L.oracle_free.argtypes = [vp]
        self.L = L

    def unit_uniform(self, seed, key, counter) -> float:
        return self.L.oracle_unit_uniform(seed, key, counter)

    GEN_KINDS = {"poisson2d": 0, "poisson27": 1, "rmat": 2}

    def gen_edges(self, kind: str, size: int, seed: int = 0):
        """Harness generator edge list (a < b, w) of a BASELINE config the
        reference has no generator for: poisson2d(size), poisson27(size, seed),
        rmat(scale=size, ef 16, seed). Returns (n, a, b, w)."""
        pa, pb, pw = C.POINTER(i32)(), C.POINTER(i32)(), C.POINTER(f64)()
        n = i32()
        m = self.L.oracle_gen_edges(self.GEN_KINDS[kind], size, seed, C.byref(pa), C.byref(pb), C.byref(pw),
                                    C.byref(n))
        out = [np.ctypeslib.as_array(p, shape=(max(m, 1),))[:m].copy() for p in (pa, pb, pw)]
        for p in (pa, pb, pw):
            self.L.oracle_free(C.cast(p, vp))
        return n.value, out[0], out[1], out[2]

    def derive_seed(self, seed, salt) -> int:
        return self.L.oracle_derive_seed(seed, salt)

    def factor(self, graph, perm, seed: int, exact: bool = False):
        """factor_randomized on (graph CSR, perm). Returns dict of arrays."""
        perm = np.ascontiguousarray(perm, np.int32)
        f = OracleFactor()
        rc = self.L.oracle_factor_randomized(graph.n, _p(graph.ptr), _p(graph.adj), _p(graph.w),
                                             _p(perm), seed, int(exact), C.byref(f))
        assert rc == 0
        n = f.n
        z = f.col_ptr[n]
        out = {
            "n": n,
            "col_ptr": np.ctypeslib.as_array(f.col_ptr, shape=(n + 1,)).copy(),
            "rows": np.ctypeslib.as_array(f.rows, shape=(max(z, 1),))[:z].copy(),
            "values": np.ctypeslib.as_array(f.values, shape=(max(z, 1),))[:z].copy(),
            "diag": np.ctypeslib.as_array(f.diag, shape=(max(n, 1),))[:n].copy(),
            "merged_degree": np.ctypeslib.as_array(f.merged_degree, shape=(max(n, 1),))[:n].copy(),
            "samples_emitted": np.ctypeslib.as_array(f.samples_emitted, shape=(max(n, 1),))[:n].copy(),
            "fills_received": np.ctypeslib.as_array(f.fills_received, shape=(max(n, 1),))[:n].copy(),
            "total_fills": f.total_fills,
            "perm": perm.copy(),
        }
        self.L.oracle_factor_free(C.byref(f))
        return out

    def checksum(self, f) -> int:
        return self.L.oracle_checksum(f["n"], _p(f["col_ptr"]), _p(f["rows"]), _p(f["values"]),
                                      _p(f["diag"]))

    def schedule_levels(self, f):
        lv = np.empty(max(f["n"], 1), np.int32)
        d = self.L.oracle_schedule_levels(f["n"], _p(f["col_ptr"]), _p(f["rows"]), _p(lv))
        return lv[:f["n"]], d

    def apply_preconditioner(self, f, r):
        r = np.ascontiguousarray(r, np.float64)
        z = np.empty(f["n"], np.float64)
        self.L.oracle_apply_preconditioner(f["n"], _p(f["col_ptr"]), _p(f["rows"]), _p(f["values"]),
                                           _p(f["diag"]), _p(f["perm"]), _p(r), _p(z))
        return z

    def laplacian_apply(self, g, x):
        x = np.ascontiguousarray(x, np.float64)
        y = np.empty(g.n, np.float64)
        self.L.oracle_laplacian_apply(g.n, _p(g.ptr), _p(g.adj), _p(g.w), _p(x), _p(y))
        return y

    def make_rhs(self, g, mode: int, seed: int):
        out = np.empty(g.n, np.float64)
        self.L.oracle_make_rhs(g.n, _p(g.ptr), _p(g.adj), _p(g.w), mode, seed, _p(out))
        return out

    def pcg(self, g, f, b, tol=1e-6, max_iters=1000):
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(g.n, np.float64)
        it, conv = C.c_int(), C.c_int()
        rel, rec = f64(), f64()
        rc = self.L.oracle_pcg(g.n, _p(g.ptr), _p(g.adj), _p(g.w), _p(f["col_ptr"]), _p(f["rows"]),
                               _p(f["values"]), _p(f["diag"]), _p(f["perm"]), _p(b), tol, max_iters,
                               _p(x), C.byref(it), C.byref(rel), C.byref(rec), C.byref(conv))
        return rc, x, {"iterations": it.value, "relative_residual": rel.value,
                       "recurrence_residual": rec.value, "converged": bool(conv.value)}


class Reference:
    """ctypes view of the unmodified reference (oracle/_ref/libparac_ref.so)."""

    SEQ, LEFT, RIGHT, EXACT = 0, 1, 2, 3

    def __init__(self, path: str = REF_LIB):
        L = C.CDLL(path)
        L.pref_last_error.restype = C.c_char_p
        L.pref_unit_uniform.restype = f64
        L.pref_unit_uniform.argtypes = [u64, i64, u64]
        L.pref_derive_seed.restype = u64
        L.pref_derive_seed.argtypes = [u64, u64]
        L.pref_graph_from_edges.argtypes = [i32, i64, vp, vp, vp, C.POINTER(vp)]
        L.pref_graph_poisson3d.argtypes = [i32, C.c_int, f64, f64, u64, C.POINTER(vp)]
        L.pref_graph_random_connected.argtypes = [i32, i64, u64, C.c_int, C.POINTER(vp)]
        L.pref_graph_random_components.argtypes = [i32, i32, i64, u64, C.POINTER(vp)]
        L.pref_graph_free.argtypes = [vp]
        L.pref_graph_n.argtypes = [vp]
        L.pref_graph_nnz.argtypes = [vp]
        L.pref_graph_nnz.restype = i64
        L.pref_graph_csr.argtypes = [vp, vp, vp, vp, vp]
        L.pref_connected_components.argtypes = [vp, vp, C.POINTER(i32)]
        L.pref_ordering_random.argtypes = [i32, u64, vp]
        L.pref_ordering_nnz_sort.argtypes = [vp, u64, vp]
        L.pref_dependency_counts.argtypes = [vp, vp, vp]
        L.pref_factor.argtypes = [vp, vp, u64, C.c_int, C.c_int, i64, i64, C.c_int,
                                  C.POINTER(f64), C.POINTER(vp)]
        L.pref_factor_left_trace.argtypes = [vp, vp, u64, C.c_int, i32, vp, C.c_int,
                                             C.POINTER(C.c_int), C.POINTER(vp)]
        L.pref_factor_free.argtypes = [vp]
        L.pref_factor_n.argtypes = [vp]
        L.pref_factor_nnz_off.argtypes = [vp]
        L.pref_factor_nnz_off.restype = i64
        L.pref_factor_copy.argtypes = [vp, vp, vp, vp, vp, vp]
        L.pref_factor_stats.argtypes = [vp, vp, vp, vp, C.POINTER(i64), C.POINTER(f64)]
        L.pref_factor_checksum.argtypes = [vp]
        L.pref_factor_checksum.restype = u64
        L.pref_factor_from_arrays.argtypes = [i32, vp, vp, vp, vp, vp, C.POINTER(vp)]
        L.pref_schedule_levels.argtypes = [vp, vp]
        L.pref_schedule_depth.argtypes = [vp]
        L.pref_apply_preconditioner.argtypes = [vp, vp, vp]
        L.pref_laplacian_apply.argtypes = [vp, vp, vp]
        L.pref_make_rhs.argtypes = [vp, C.c_int, u64, vp]
        L.pref_pcg.argtypes = [vp, vp, vp, f64, C.c_int, vp, C.POINTER(C.c_int), C.POINTER(f64),
                               C.POINTER(f64), C.POINTER(C.c_int), C.POINTER(f64)]
        L.pref_read_laplacian.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.pref_write_matrix_market.argtypes = [C.c_char_p, vp]
        L.pref_write_factor.argtypes = [vp, C.c_char_p]
        L.pref_read_factor.argtypes = [C.c_char_p, C.c_char_p, C.POINTER(vp)]
        L.pref_write_vector.argtypes = [C.c_char_p, i64, vp]
        L.pref_read_vector.argtypes = [C.c_char_p, i64, vp, C.POINTER(i64)]
        L.pref_write_permutation.argtypes = [C.c_char_p, i32, vp]
        self.L = L

    @staticmethod
    def available(path: str = REF_LIB) -> bool:
        return os.path.exists(path)

    def _chk(self, rc):
        if rc != 0:
            raise RuntimeError(f"reference error {rc}: {self.L.pref_last_error().decode()}")

    # graphs (handles)
    def graph_from_csr(self, g):
        """Rebuild a reference LaplacianGraph from a CSR (lower triplets)."""
        src = np.repeat(np.arange(g.n, dtype=np.int32), np.diff(g.ptr))
        lower = g.adj > src
        a = np.ascontiguousarray(src[lower]); b = np.ascontiguousarray(g.adj[lower])
        w = np.ascontiguousarray(g.w[lower])
        h = vp()
        self._chk(self.L.pref_graph_from_edges(g.n, len(a), _p(a), _p(b), _p(w), C.byref(h)))
        return h

    def graph_from_edges(self, n, a, b, w):
        """LaplacianGraph::from_edges (src/graph.cpp:21) of an edge list."""
        a, b = np.ascontiguousarray(a, np.int32), np.ascontiguousarray(b, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        h = vp()
        self._chk(self.L.pref_graph_from_edges(n, len(a), _p(a), _p(b), _p(w), C.byref(h)))
        return h

    def workload_graph(self, workload: str, seed: int = 0):
        """Reference LaplacianGraph of a bench.py workload, built without the
        product library: gen_poisson3d through the reference itself, the other
        configs from the port's harness generators + the reference's from_edges."""
        kind = {"poisson3d_128": ("p3", 128), "batch_64x64": ("p3", 64), "poisson2d_256": ("poisson2d", 256),
                "poisson27_96": ("poisson27", 96), "rmat_22": ("rmat", 22)}[workload]
        if kind[0] == "p3":
            return self.poisson3d(kind[1])
        n, a, b, w = Port().gen_edges(kind[0], kind[1], 1 if kind[0] == "poisson27" else seed)
        return self.graph_from_edges(n, a, b, w)

    def poisson3d(self, n, variant=0, eps=1e-3, contrast=1e4, seed=0):
        h = vp()
        self._chk(self.L.pref_graph_poisson3d(n, variant, eps, contrast, seed, C.byref(h)))
        return h

    def random_connected(self, n, extra, seed, unit=False):
        h = vp()
        self._chk(self.L.pref_graph_random_connected(n, extra, seed, int(unit), C.byref(h)))
        return h

    def random_components(self, n, comps, extra, seed):
        h = vp()
        self._chk(self.L.pref_graph_random_components(n, comps, extra, seed, C.byref(h)))
        return h

    def csr(self, h):
        n = self.L.pref_graph_n(h)
        nnz = self.L.pref_graph_nnz(h)
        ptr = np.empty(n + 1, np.int64); adj = np.empty(max(nnz, 1), np.int32)
        w = np.empty(max(nnz, 1), np.float64); wdeg = np.empty(max(n, 1), np.float64)
        self.L.pref_graph_csr(h, _p(ptr), _p(adj), _p(w), _p(wdeg))
        return n, ptr, adj[:nnz], w[:nnz], wdeg[:n]

    def ordering_random(self, n, seed):
        p = np.empty(n, np.int32)
        self._chk(self.L.pref_ordering_random(n, seed, _p(p)))
        return p

    def ordering_nnz_sort(self, h, seed):
        p = np.empty(self.L.pref_graph_n(h), np.int32)
        self._chk(self.L.pref_ordering_nnz_sort(h, seed, _p(p)))
        return p

    def factor(self, h, perm, seed, backend=0, workers=1, arena=-1, workspace=-1, stats=False):
        perm = np.ascontiguousarray(perm, np.int32)
        f = vp()
        wall = f64()
        self._chk(self.L.pref_factor(h, _p(perm), seed, backend, workers, arena, workspace,
                                     int(stats), C.byref(wall), C.byref(f)))
        return f, wall.value

    def factor_arrays(self, f):
        n = self.L.pref_factor_n(f)
        z = self.L.pref_factor_nnz_off(f)
        out = {"n": n, "col_ptr": np.empty(n + 1, np.int64), "rows": np.empty(max(z, 1), np.int32),
               "values": np.empty(max(z, 1), np.float64), "diag": np.empty(max(n, 1), np.float64),
               "perm": np.empty(max(n, 1), np.int32)}
        self.L.pref_factor_copy(f, _p(out["col_ptr"]), _p(out["rows"]), _p(out["values"]),
                                _p(out["diag"]), _p(out["perm"]))
        for k in ("rows", "values"):
            out[k] = out[k][:z]
        for k in ("diag", "perm"):
            out[k] = out[k][:n]
        return out

    def factor_stats(self, f):
        n = self.L.pref_factor_n(f)
        m, s, fl = (np.empty(max(n, 1), np.int32) for _ in range(3))
        tf, sec = i64(), f64()
        assert self.L.pref_factor_stats(f, _p(m), _p(s), _p(fl), C.byref(tf), C.byref(sec)) == 0
        return {"merged_degree": m[:n], "samples_emitted": s[:n], "fills_received": fl[:n],
                "total_fills": tf.value, "seconds": sec.value}

    def checksum(self, f) -> int:
        return self.L.pref_factor_checksum(f)

    def make_rhs(self, h, mode: int, seed: int):
        out = np.empty(self.L.pref_graph_n(h), np.float64)
        self._chk(self.L.pref_make_rhs(h, mode, seed, _p(out)))
        return out

    def pcg(self, h, f, b, tol=1e-8, max_iters=1000):
        """pcg_solve (src/solver.cpp:95-175) through the reference's public API;
        `seconds` is its own SolveReport::solve_seconds."""
        b = np.ascontiguousarray(b, np.float64)
        x = np.empty(len(b), np.float64)
        it, conv = C.c_int(), C.c_int()
        rel, rec, sec = f64(), f64(), f64()
        self._chk(self.L.pref_pcg(h, f, _p(b), tol, max_iters, _p(x), C.byref(it), C.byref(rel), C.byref(rec),
                                  C.byref(conv), C.byref(sec)))
        return x, {"iterations": it.value, "relative_residual": rel.value, "recurrence_residual": rec.value,
                   "converged": bool(conv.value), "seconds": sec.value}

    def free_factor(self, f):
        self.L.pref_factor_free(f)

    def free_graph(self, h):
        self.L.pref_graph_free(h)
