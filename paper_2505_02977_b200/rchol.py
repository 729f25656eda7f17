"""Host-side mirror of the reference's public interface for the rchol hot path.

Names, argument meaning and error behaviour follow the reference library
`parac` (/root/reference/proj/include/parac/*.hpp) so parity tests read like the
reference's own tests:

  LaplacianGraph        graph.hpp:25-60      (CSR, neighbours ascending)
  Ordering              ordering.hpp:13-24   (perm: label -> position)
  LdlFactor             factor.hpp:18-32     (same_values, checksum, nnz)
  FactorStats           factor_seq.hpp:22-30
  GpuOptions            factor_par.hpp:31-45 (ParOptions analogue)
  factor_gpu            factor_par.hpp:53-62 (factor_parallel_left/right drop-in)
  pcg_solve_gpu         solver.hpp:39-42
  apply_preconditioner_gpu / laplacian_apply_gpu   solver.hpp:30,33
  Error / Errc          error.hpp:9-40

Everything computes through the CUDA library (lib/libparac_gpu.so); numpy is
only the host container.
"""
from __future__ import annotations

import ctypes as C
import time
import os
import enum
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib as L

lib = L.lib


class Errc(enum.IntEnum):
    """parac::Errc (include/parac/error.hpp:9-27), same numbering."""
    asymmetric_input = 1
    positive_off_diagonal = 2
    row_sum_violation = 3
    too_large_for_dense = 4
    parse_error = 5
    unsupported_field = 6
    budget_exceeded = 7
    not_a_permutation = 8
    dense_blowup = 9
    arena_exhausted = 10
    queue_stall = 11
    workspace_full = 12
    dimension_mismatch = 13
    not_connected = 14
    too_many_neighbors = 15
    io_error = 16
    internal_error = 17


class Error(RuntimeError):
    """parac::Error: carries an Errc code; message is "<ErrcName>: detail"."""

    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = Errc(code)


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib.parac_gpu_last_error().decode(errors="replace")
        raise Error(rc, msg)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# --------------------------------------------------------------------- graph
class LaplacianGraph:
    """Immutable weighted graph of a Laplacian (graph.hpp:25-60), label space."""

    def __init__(self, n: int, ptr: np.ndarray, adj: np.ndarray, w: np.ndarray,
                 wdeg: Optional[np.ndarray] = None):
        self.n = int(n)
        self.ptr = np.ascontiguousarray(ptr, dtype=np.int64)
        self.adj = np.ascontiguousarray(adj, dtype=np.int32)
        self.w = np.ascontiguousarray(w, dtype=np.float64)
        if wdeg is None:
            wdeg = np.array([float(sum(self.w[self.ptr[v]:self.ptr[v + 1]].tolist()))
                             for v in range(self.n)], dtype=np.float64)
        self.wdeg = wdeg

    @staticmethod
    def _from_native(g: "L.parac_graph") -> "LaplacianGraph":
        n, nnz = g.n, g.nnz
        ptr = np.ctypeslib.as_array(g.ptr, shape=(n + 1,)).copy()
        adj = np.ctypeslib.as_array(g.adj, shape=(max(nnz, 1),))[:nnz].copy()
        w = np.ctypeslib.as_array(g.w, shape=(max(nnz, 1),))[:nnz].copy()
        wdeg = np.ctypeslib.as_array(g.wdeg, shape=(max(n, 1),))[:n].copy()
        lib.parac_graph_free(C.byref(g))
        return LaplacianGraph(n, ptr, adj, w, wdeg)

    @staticmethod
    def from_edges(n: int, edges: Sequence) -> "LaplacianGraph":
        """LaplacianGraph::from_edges (src/graph.cpp:21-83); edges = [(a, b, w), ...]."""
        e = list(edges)
        a = np.array([x[0] for x in e], dtype=np.int32)
        b = np.array([x[1] for x in e], dtype=np.int32)
        w = np.array([x[2] for x in e], dtype=np.float64)
        g = L.parac_graph()
        _check(lib.parac_graph_from_edges(n, len(e), _ptr(a), _ptr(b), _ptr(w), C.byref(g)))
        return LaplacianGraph._from_native(g)

    def num_vertices(self) -> int:
        return self.n

    def num_edges(self) -> int:
        return int(self.ptr[self.n]) // 2

    nnz_lower = num_edges

    def nnz_off_diagonal(self) -> int:
        return int(self.ptr[self.n])

    def degree(self, v: int) -> int:
        return int(self.ptr[v + 1] - self.ptr[v])

    def neighbors(self, v: int) -> np.ndarray:
        return self.adj[self.ptr[v]:self.ptr[v + 1]]

    def weights(self, v: int) -> np.ndarray:
        return self.w[self.ptr[v]:self.ptr[v + 1]]

    def weighted_degree(self, v: int) -> float:
        return float(self.wdeg[v])

    def csr(self) -> "L.parac_csr":
        return L.parac_csr(self.n, _ptr(self.ptr), _ptr(self.adj), _ptr(self.w))


def _gen(fn, *args) -> LaplacianGraph:
    g = L.parac_graph()
    _check(fn(*args, C.byref(g)))
    return LaplacianGraph._from_native(g)


def gen_poisson3d(n: int, variant: str = "uniform", epsilon: float = 1e-3,
                  contrast_ratio: float = 1e4, seed: int = 0) -> LaplacianGraph:
    """gen_poisson3d (generators.hpp:26); variant uniform|anisotropic|contrast."""
    v = {"uniform": 0, "anisotropic": 1, "contrast": 2}[variant]
    return _gen(lib.parac_gen_poisson3d, n, v, epsilon, contrast_ratio, seed)


def gen_poisson2d(n: int) -> LaplacianGraph:
    return _gen(lib.parac_gen_poisson2d, n)


def gen_poisson27(n: int, seed: int = 1) -> LaplacianGraph:
    return _gen(lib.parac_gen_poisson27, n, seed)


def gen_rmat(scale: int, edge_factor: int = 16, seed: int = 0) -> LaplacianGraph:
    return _gen(lib.parac_gen_rmat, scale, edge_factor, seed)


def gen_random_connected(n: int, extra_edges: int, seed: int,
                         unit_weights: bool = False) -> LaplacianGraph:
    return _gen(lib.parac_gen_random_connected, n, extra_edges, seed, int(unit_weights))


def gen_random_components(n: int, components: int, extra_edges: int,
                          seed: int) -> LaplacianGraph:
    return _gen(lib.parac_gen_random_components, n, components, extra_edges, seed)


# ------------------------------------------------------------------ ordering
class Ordering:
    """perm[label] = position; inverse[position] = label (ordering.hpp:13-24)."""

    def __init__(self, perm: np.ndarray):
        perm = np.ascontiguousarray(perm, dtype=np.int32)
        _check(lib.parac_ordering_check(len(perm), _ptr(perm)))
        self.perm = perm
        self.inverse = np.empty_like(perm)
        self.inverse[perm] = np.arange(len(perm), dtype=np.int32)

    @staticmethod
    def identity(n: int) -> "Ordering":
        return Ordering(np.arange(n, dtype=np.int32))

    from_positions = staticmethod(lambda positions: Ordering(np.asarray(positions)))

    def size(self) -> int:
        return len(self.perm)


def ordering_random(n: int, seed: int) -> Ordering:
    perm = np.empty(n, dtype=np.int32)
    _check(lib.parac_ordering_random(n, seed, _ptr(perm)))
    return Ordering(perm)


def ordering_nnz_sort(graph: LaplacianGraph, seed: int) -> Ordering:
    perm = np.empty(graph.n, dtype=np.int32)
    csr = graph.csr()
    _check(lib.parac_ordering_nnz_sort(C.byref(csr), seed, _ptr(perm)))
    return Ordering(perm)


# -------------------------------------------------------------------- factor
@dataclass
class FactorStats:
    """FactorStats (factor_seq.hpp:22-30) plus device timings."""
    merged_degree: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    samples_emitted: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    fills_received: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    total_fills: int = 0
    arena_used: int = 0
    fill_pool_used: int = 0
    max_raw: int = 0
    large_columns: int = 0
    seconds: float = 0.0
    setup_ms: float = 0.0
    eliminate_ms: float = 0.0
    assemble_ms: float = 0.0
    device_ms: float = 0.0
    upload_ms: float = 0.0
    attempts: int = 0


@dataclass
class GpuOptions:
    """ParOptions analogue (factor_par.hpp:31-45)."""
    fill_pool_entries: int = -1      # arena_budget analogue; <0 = default (grows on retry)
    column_arena_entries: int = -1
    first_chunk: int = 0
    watchdog_seconds: float = 60.0
    record_stats: bool = True
    verify: bool = False             # TestHooks::verify analogue (device assertions)
    grid_ctas: int = 0
    delay_ns: int = 0                # TestHooks::delay analogue (random __nanosleep)
    record_times: bool = False       # ParOptions::record_vertex_times analogue
    trace_position: int = -1         # TestHooks::on_phase analogue: >= 0 snapshots dp for this position

    def native(self) -> "L.parac_gpu_options":
        o = L.parac_gpu_options()
        lib.parac_gpu_default_options(C.byref(o))
        o.fill_pool_entries = self.fill_pool_entries
        o.column_arena_entries = self.column_arena_entries
        o.first_chunk = self.first_chunk
        o.watchdog_seconds = self.watchdog_seconds
        o.record_stats = int(self.record_stats)
        o.verify = int(self.verify)
        o.grid_ctas = self.grid_ctas
        o.delay_ns = self.delay_ns
        o.record_times = int(self.record_times)
        o.trace_phases = int(self.trace_position >= 0)
        o.trace_position = max(self.trace_position, 0)
        return o


class LdlFactor:
    """LdlFactor (factor.hpp:18-32): unit-lower G in CSC + D, position space."""

    def __init__(self, n, col_ptr, rows, values, diag, perm):
        self.n = int(n)
        self.col_ptr = np.ascontiguousarray(col_ptr, dtype=np.int64)
        self.rows = np.ascontiguousarray(rows, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        self.diag = np.ascontiguousarray(diag, dtype=np.float64)
        self.perm = np.ascontiguousarray(perm, dtype=np.int32)

    def nnz_off_diagonal(self) -> int:
        return len(self.rows)

    def nnz(self) -> int:
        return len(self.rows) + self.n

    def same_values(self, other: "LdlFactor") -> bool:
        """Byte identity of every array (src/factor.cpp:10-13)."""
        return (self.n == other.n and np.array_equal(self.col_ptr, other.col_ptr)
                and np.array_equal(self.rows, other.rows)
                and self.values.tobytes() == other.values.tobytes()
                and self.diag.tobytes() == other.diag.tobytes()
                and np.array_equal(self.perm, other.perm))

    def checksum(self) -> int:
        return int(lib.parac_factor_checksum(self.n, _ptr(self.col_ptr), _ptr(self.rows),
                                             _ptr(self.values), _ptr(self.diag)))


class GpuContext:
    """Owns a device context (buffers + stream) of the C ABI."""

    def __init__(self, device: int = 0):
        h = C.c_void_p()
        _check(lib.parac_gpu_create(device, C.byref(h)))
        self.handle = h
        self.device = device
        self._graph = None
        self._factor_n = -1
        # the LdlFactor object whose arrays are the context's resident factor
        # (factors are immutable inputs, like the reference's const LdlFactor&;
        # the ones factor_gpu returns are marked read-only)
        self._resident = None

    def close(self) -> None:
        if self.handle:
            lib.parac_gpu_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- staging
    def upload(self, graph: LaplacianGraph, ordering: Ordering) -> None:
        if ordering.size() != graph.n:
            raise Error(Errc.dimension_mismatch, "DimensionMismatch: ordering size does not match graph")
        csr = graph.csr()
        _check(lib.parac_gpu_upload(self.handle, C.byref(csr), _ptr(ordering.perm)))
        self._graph = (graph, ordering)
        self._resident = None  # staging a graph drops the resident factor

    def factor_resident(self, seed: int, options: Optional[GpuOptions] = None):
        o = (options or GpuOptions()).native()
        info = L.parac_gpu_factor_info()
        _check(lib.parac_gpu_factor_resident(self.handle, seed, C.byref(o), C.byref(info)))
        self._factor_n = info.n
        self._resident = None
        return info

    def factor_to_host(self, seed: int, options: Optional[GpuOptions] = None, out=None,
                       capacity: Optional[int] = None):
        """parac_gpu_factor_begin + parac_gpu_factor_end on the staged input:
        the factor is copied to host arrays while it is computed (each column
        as soon as it and every column before it are final). out = (col_ptr,
        rows, values, diag) host arrays (pinned or pageable), default fresh
        numpy arrays sized from the last factor of this context or capacity.
        Returns (info, out); raises Error(budget_exceeded)
        when Z exceeds the capacity (the factor stays resident)."""
        graph, _ = self._graph
        n = graph.n
        o = (options or GpuOptions()).native()
        if out is None:
            cap = capacity if capacity is not None else 0
            out = (np.empty(n + 1, np.int64), np.empty(max(cap, 1), np.int32),
                   np.empty(max(cap, 1), np.float64), np.empty(max(n, 1), np.float64))
        cap = capacity if capacity is not None else len(out[1])
        info = L.parac_gpu_factor_info()
        _check(lib.parac_gpu_factor_begin(self.handle, seed, C.byref(o)))
        self._factor_n = -1
        self._resident = None
        rc = lib.parac_gpu_factor_end(self.handle, C.byref(info), *[_ptr(a) for a in out], cap)
        if rc in (0, int(Errc.budget_exceeded)):
            self._factor_n = info.n
        _check(rc)
        return info, out

    def download(self, with_stats: bool = True):
        graph, ordering = self._graph
        n = graph.n
        col_ptr = np.empty(n + 1, np.int64)
        _check(lib.parac_gpu_download(self.handle, _ptr(col_ptr), None, None, None, None, None, None))
        z = int(col_ptr[n])
        rows = np.empty(max(z, 1), np.int32)
        vals = np.empty(max(z, 1), np.float64)
        diag = np.empty(max(n, 1), np.float64)
        st = [np.empty(max(n, 1), np.int32) for _ in range(3)] if with_stats else [None] * 3
        _check(lib.parac_gpu_download(self.handle, _ptr(col_ptr), _ptr(rows), _ptr(vals),
                                      _ptr(diag), *[(_ptr(a) if a is not None else None) for a in st]))
        f = LdlFactor(n, col_ptr, rows[:z], vals[:z], diag[:n], ordering.perm)
        return f, [a[:n] if a is not None else None for a in st]

    def vertex_times(self) -> np.ndarray:
        """[n, 8] phase timestamps (globaltimer ns) per position (record_times runs);
        column 0 = start, 7 = end; see parac_gpu_download_times."""
        n = self._factor_n
        out = np.empty(8 * max(n, 1), np.uint64)
        _check(lib.parac_gpu_download_times(self.handle, _ptr(out)))
        return out[:8 * n].reshape(n, 8)

    PHASES = ("gathered", "sampled", "decremented")  # TestHooks::Phase (factor_par.hpp:17)

    def phase_snapshots(self) -> dict:
        """TestHooks::on_phase analogue of the last run with trace_position set:
        {phase: dp snapshot (int64[n])} for each phase the traced position
        reached (parac_gpu_download_phase_snapshots)."""
        n = self._factor_n
        dp = np.empty(3 * max(n, 1), np.int64)
        taken = np.zeros(3, np.int32)
        _check(lib.parac_gpu_download_phase_snapshots(self.handle, _ptr(dp), _ptr(taken)))
        return {ph: dp[i * n:(i + 1) * n].copy() for i, ph in enumerate(self.PHASES) if taken[i]}

    PRECOND_MODES = {"default": 0, "exact": 1, "fast": 2}

    def set_preconditioner_mode(self, mode: str) -> None:
        """'default' (apply exact, pcg fast), 'exact' or 'fast'; see parac_gpu.h."""
        _check(lib.parac_gpu_set_preconditioner_mode(self.handle, self.PRECOND_MODES[mode]))

    def upload_factor(self, f: LdlFactor) -> None:
        self._resident = None  # the previous resident factor is dropped even if f is rejected
        _check(lib.parac_gpu_upload_factor(self.handle, f.n, _ptr(f.col_ptr), _ptr(f.rows),
                                           _ptr(f.values), _ptr(f.diag), _ptr(f.perm)))
        self._factor_n = f.n
        self._resident = f

    def ensure_factor(self, f: LdlFactor) -> None:
        """Make f the resident factor; no copy when it already is (same object)."""
        if self._resident is not f:
            self.upload_factor(f)


_default_ctx: Optional[GpuContext] = None


def default_context() -> GpuContext:
    global _default_ctx
    if _default_ctx is None:
        _default_ctx = GpuContext(0)
    return _default_ctx


def device_count() -> int:
    return int(lib.parac_gpu_device_count())


def factor_gpu(graph: LaplacianGraph, ordering: Ordering, seed: int,
               options: Optional[GpuOptions] = None, stats: Optional[FactorStats] = None,
               ctx: Optional[GpuContext] = None) -> LdlFactor:
    """Drop-in for factor_parallel_left (factor_par.hpp:53-55): byte-identical
    LdlFactor to factor_randomized for the same graph, ordering and seed."""
    t0 = time.perf_counter()
    ctx = ctx or default_context()
    ctx.upload(graph, ordering)
    n = graph.n
    # the factor is copied out while it is computed (parac_gpu_factor_end):
    # outputs are sized by a bound on Z -- np.empty only reserves address
    # space, pages are touched by the copy -- and a factor beyond the bound
    # is fetched afterwards from the resident copy
    cap = 4 * graph.nnz_off_diagonal() + n + 1024
    out = (np.empty(n + 1, np.int64), np.empty(cap, np.int32), np.empty(cap, np.float64),
           np.empty(max(n, 1), np.float64))
    info = L.parac_gpu_factor_info()
    _check(lib.parac_gpu_factor_begin(ctx.handle, seed, C.byref((options or GpuOptions()).native())))
    ctx._factor_n = -1
    ctx._resident = None
    rc = lib.parac_gpu_factor_end(ctx.handle, C.byref(info), *[_ptr(a) for a in out], cap)
    if rc not in (0, int(Errc.budget_exceeded)):
        _check(rc)
    ctx._factor_n = info.n
    if rc == 0:
        z = info.nnz_off_diagonal
        f = LdlFactor(n, out[0], out[1][:z], out[2][:z], out[3][:n], ordering.perm)
        st = [None] * 3
        if stats is not None:
            st = [np.empty(max(n, 1), np.int32) for _ in range(3)]
            _check(lib.parac_gpu_download(ctx.handle, None, None, None, None, *[_ptr(a) for a in st]))
            st = [a[:n] for a in st]
    else:  # a factor beyond the bound: fetch it from the resident copy
        f, st = ctx.download(with_stats=stats is not None)
    for a in (f.col_ptr, f.rows, f.values, f.diag):
        a.flags.writeable = False
    ctx._resident = f  # the device copy stays resident for solves on this factor
    if stats is not None:
        stats.merged_degree, stats.samples_emitted, stats.fills_received = st
        stats.total_fills = info.total_fills
        stats.arena_used = info.arena_used
        stats.fill_pool_used = info.fill_pool_used
        stats.max_raw = info.max_raw
        stats.large_columns = info.large_columns
        stats.setup_ms = info.setup_ms
        stats.eliminate_ms = info.eliminate_ms
        stats.assemble_ms = info.assemble_ms
        stats.device_ms = info.device_ms
        stats.upload_ms = info.upload_ms
        stats.attempts = info.attempts
        # FactorStats::seconds is wall time at the API, as in the reference
        # (factor_seq.cpp:46, factor_par.cpp); device_ms holds the device time
        stats.seconds = time.perf_counter() - t0
    return f


def _batch_args(graphs, orderings, seeds):
    if not (len(graphs) == len(orderings) == len(seeds)) or not graphs:
        raise Error(Errc.dimension_mismatch, "DimensionMismatch: batch lists differ in length")
    for g, o in zip(graphs, orderings):
        if o.size() != g.n:
            raise Error(Errc.dimension_mismatch, "DimensionMismatch: ordering size does not match graph")
    csrs = (L.parac_csr * len(graphs))(*[g.csr() for g in graphs])
    perms = (C.c_void_p * len(graphs))(*[_ptr(o.perm) for o in orderings])
    sd = np.ascontiguousarray(seeds, dtype=np.uint64)
    keep = (csrs, perms, sd, graphs, orderings)
    return csrs, perms, sd, keep


def factor_batch_gpu(graphs: Sequence[LaplacianGraph], orderings: Sequence[Ordering], seeds: Sequence[int],
                     options: Optional[GpuOptions] = None, ctx: Optional[GpuContext] = None):
    """Factor independent Laplacians in ONE device pass (BASELINE config[4]): the
    problems are staged as a disjoint union with per-problem sample seeds and
    keys, so factor i is byte-identical to factor_gpu(graphs[i], orderings[i],
    seeds[i]). Returns (list of LdlFactor, info)."""
    ctx = ctx or default_context()
    csrs, perms, sd, keep = _batch_args(graphs, orderings, seeds)
    o = (options or GpuOptions()).native()
    info = L.parac_gpu_factor_info()
    k = len(graphs)
    # every member copied out while the union is factored
    # (parac_gpu_factor_batch_to_host); rows/values sized by a bound on each
    # member's Z (address space only), a larger member fetched afterwards
    caps = np.array([4 * g.nnz_off_diagonal() + g.n + 1024 for g in graphs], np.int64)
    bufs = [(np.empty(g.n + 1, np.int64), np.empty(int(c), np.int32), np.empty(int(c), np.float64),
             np.empty(max(g.n, 1), np.float64)) for g, c in zip(graphs, caps)]
    arr = [(C.c_void_p * k)(*[_ptr(b[j]) for b in bufs]) for j in range(4)]
    rc = lib.parac_gpu_factor_batch_to_host(ctx.handle, k, csrs, perms, _ptr(sd), C.byref(o), C.byref(info),
                                            *arr, _ptr(caps))
    if rc not in (0, int(Errc.budget_exceeded)):
        _check(rc)
    ctx._factor_n = info.n
    ctx._graph = None      # the context now holds the batch union,
    ctx._resident = None   # not any single graph or factor
    out = []
    for i, (g, ordg, b) in enumerate(zip(graphs, orderings, bufs)):
        z = C.c_int64()
        _check(lib.parac_gpu_batch_nnz(ctx.handle, i, C.byref(z)))
        z = int(z.value)
        col_ptr, rows, vals, diag = b
        if z > caps[i]:
            rows = np.empty(max(z, 1), np.int32)
            vals = np.empty(max(z, 1), np.float64)
            _check(lib.parac_gpu_download_batch(ctx.handle, i, _ptr(col_ptr), _ptr(rows), _ptr(vals), _ptr(diag)))
        out.append(LdlFactor(g.n, col_ptr, rows[:z], vals[:z], diag[:g.n], ordg.perm))
    del keep
    return out, info


def dependency_counts(graph: LaplacianGraph, ordering: Ordering) -> np.ndarray:
    """dependency_counts (factor_seq.hpp:45-46): earlier-neighbour count per position."""
    pos = ordering.perm
    out = np.zeros(graph.n, np.int32)
    src = np.repeat(np.arange(graph.n), np.diff(graph.ptr))
    earlier = pos[graph.adj] < pos[src]
    np.add.at(out, pos[src[earlier]], 1)
    return out


# --------------------------------------------------------------------- solve
@dataclass
class SolveConfig:
    tol: float = 1e-6
    max_iters: int = 1000


@dataclass
class SolveReport:
    iterations: int = 0
    relative_residual: float = 0.0
    recurrence_residual: float = 0.0
    converged: bool = False
    factor_seconds: float = 0.0
    solve_seconds: float = 0.0
    device_ms: float = 0.0
    exact: bool = False  # the bit-exact PCG ran (x and this report are the reference's bytes)


def _stage_for_solve(ctx: GpuContext, graph: Optional[LaplacianGraph], factor: LdlFactor):
    if graph is not None:
        g_cur = ctx._graph[0] if ctx._graph else None
        if g_cur is not graph:
            ctx.upload(graph, Ordering(factor.perm))
    ctx.ensure_factor(factor)


def pcg_solve_gpu(graph: LaplacianGraph, factor: LdlFactor, b: np.ndarray,
                  config: Optional[SolveConfig] = None, ctx: Optional[GpuContext] = None):
    """pcg_solve (solver.hpp:39-42) on the device. Returns (x, SolveReport)."""
    config = config or SolveConfig()
    ctx = ctx or default_context()
    if len(b) != graph.n or factor.n != graph.n:
        raise Error(Errc.dimension_mismatch, "DimensionMismatch: solver inputs disagree on size")
    _stage_for_solve(ctx, graph, factor)
    return _pcg_resident(ctx, b, config)


def _pcg_resident(ctx: GpuContext, b: np.ndarray, config: SolveConfig):
    b = np.ascontiguousarray(b, dtype=np.float64)
    x = np.empty(len(b), np.float64)
    rep = L.parac_gpu_solve_report()
    _check(lib.parac_gpu_pcg(ctx.handle, _ptr(b), config.tol, config.max_iters, _ptr(x),
                             C.byref(rep)))
    return x, SolveReport(rep.iterations, rep.relative_residual, rep.recurrence_residual,
                          bool(rep.converged), 0.0, rep.wall_ms / 1e3, rep.solve_ms, bool(rep.exact))


def apply_preconditioner_gpu(factor: LdlFactor, r: np.ndarray,
                             ctx: Optional[GpuContext] = None) -> np.ndarray:
    """apply_preconditioner (solver.hpp:30): z = G^-T D^+ G^-1 r in label space."""
    ctx = ctx or default_context()
    if len(r) != factor.n:
        raise Error(Errc.dimension_mismatch,
                    f"DimensionMismatch: vector length {len(r)} vs factor size {factor.n}")
    ctx.ensure_factor(factor)
    r = np.ascontiguousarray(r, dtype=np.float64)
    z = np.empty(factor.n, np.float64)
    _check(lib.parac_gpu_apply_preconditioner(ctx.handle, _ptr(r), _ptr(z)))
    return z


def laplacian_apply_gpu(graph: LaplacianGraph, x: np.ndarray,
                        ctx: Optional[GpuContext] = None) -> np.ndarray:
    """laplacian_apply (solver.hpp:33): y = L x, fixed per-row order."""
    ctx = ctx or default_context()
    if len(x) != graph.n:
        raise Error(Errc.dimension_mismatch,
                    f"DimensionMismatch: vector length {len(x)} vs graph size {graph.n}")
    ctx.upload(graph, Ordering.identity(graph.n))
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(graph.n, np.float64)
    _check(lib.parac_gpu_laplacian_apply(ctx.handle, _ptr(x), _ptr(y)))
    return y


def schedule_levels_gpu(factor: LdlFactor, ctx: Optional[GpuContext] = None):
    """schedule_levels / schedule_depth (factor_par.hpp:66-70). Returns (levels, depth)."""
    ctx = ctx or default_context()
    ctx.ensure_factor(factor)
    lv = np.empty(max(factor.n, 1), np.int32)
    depth = C.c_int32()
    _check(lib.parac_gpu_schedule_levels(ctx.handle, _ptr(lv), C.byref(depth)))
    return lv[:factor.n], int(depth.value)


def ordering_nnz_sort_gpu(graph: LaplacianGraph, seed: int, ctx: Optional[GpuContext] = None) -> Ordering:
    """ordering_nnz_sort (ordering.hpp:32, src/ordering.cpp:49-70) computed on the
    device: keys and a stable radix sort by (tie bits, degree); same perm as the
    reference's std::sort."""
    ctx = ctx or default_context()
    perm = np.empty(max(graph.n, 1), dtype=np.int32)
    csr = graph.csr()
    _check(lib.parac_gpu_ordering_nnz_sort(ctx.handle, C.byref(csr), seed, _ptr(perm)))
    return Ordering(perm[:graph.n])


# ------------------------------------------------- Matrix Market I/O (8(f)-4)
def _b(path) -> bytes:
    return os.fsencode(path)


def read_laplacian(path) -> LaplacianGraph:
    """read_laplacian (matrix_market.hpp:30, src/matrix_market.cpp:129-135)."""
    g = L.parac_graph()
    _check(lib.parac_read_laplacian(_b(path), C.byref(g)))
    return LaplacianGraph._from_native(g)


def write_matrix_market(path, graph: LaplacianGraph) -> None:
    """write_matrix_market (src/matrix_market.cpp:137-159), byte-identical."""
    csr = graph.csr()
    _check(lib.parac_write_matrix_market(_b(path), C.byref(csr)))


def write_factor(factor: LdlFactor, stem) -> None:
    """write_factor (src/matrix_market.cpp:161-184): <stem>.G.mtx + <stem>.D.mtx."""
    _check(lib.parac_write_factor(_b(stem), factor.n, _ptr(factor.col_ptr), _ptr(factor.rows),
                                  _ptr(factor.values), _ptr(factor.diag)))


def read_factor(stem, perm_path="") -> LdlFactor:
    """read_factor (src/matrix_market.cpp:186-266)."""
    f = L.parac_factor()
    _check(lib.parac_read_factor(_b(stem), _b(perm_path) if perm_path else None, C.byref(f)))
    try:
        n, z = f.n, f.nnz
        arr = lambda p, k: np.ctypeslib.as_array(p, shape=(max(k, 1),))[:k].copy()  # noqa: E731
        return LdlFactor(n, arr(f.col_ptr, n + 1), arr(f.rows, z), arr(f.values, z), arr(f.diag, n),
                         arr(f.perm, n))
    finally:
        lib.parac_factor_free(C.byref(f))


def write_vector(path, values) -> None:
    """write_vector (src/matrix_market.cpp:268-276)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    _check(lib.parac_write_vector(_b(path), len(v), _ptr(v)))


def read_vector(path) -> np.ndarray:
    """read_vector (src/matrix_market.cpp:278-304)."""
    p = C.POINTER(C.c_double)()
    n = C.c_int64()
    _check(lib.parac_read_vector(_b(path), C.byref(p), C.byref(n)))
    try:
        return np.ctypeslib.as_array(p, shape=(max(n.value, 1),))[:n.value].copy()
    finally:
        lib.parac_free_array(C.cast(p, C.c_void_p))


def write_permutation(path, ordering: Ordering) -> None:
    """write_permutation (src/ordering.cpp:87-93)."""
    perm = np.ascontiguousarray(ordering.perm, dtype=np.int32)
    _check(lib.parac_write_permutation(_b(path), len(perm), _ptr(perm)))


def ordering_from_file(path, n: int) -> Ordering:
    """ordering_from_file (src/ordering.cpp:72-85) + from_positions validation."""
    perm = np.empty(max(n, 1), dtype=np.int32)
    _check(lib.parac_read_permutation(_b(path), n, _ptr(perm)))
    return Ordering(perm[:n])


RHS_MODES = {"random_projected": 1, "from_random_x": 2}


def make_rhs(graph: LaplacianGraph, mode: str, seed: int) -> np.ndarray:
    """make_rhs (solver.hpp:47, src/solver.cpp:177-193), host libm like the reference."""
    out = np.empty(graph.n, np.float64)
    csr = graph.csr()
    _check(lib.parac_make_rhs(C.byref(csr), RHS_MODES[mode], seed, _ptr(out)))
    return out
