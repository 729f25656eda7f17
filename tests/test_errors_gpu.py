"""GPU: malformed inputs fail with the reference's Errc codes and leave the
context usable (no hang, no stale resident state). The reference's own
apply_preconditioner/schedule_levels would just read a malformed factor; the
device sweeps wait on earlier columns, so the C ABI validates first
(parac_gpu_upload_factor, parac_gpu_upload_batch)."""
import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import factor_from_port

pytestmark = pytest.mark.gpu


def _good(port):
    g = P.gen_poisson3d(6)
    o = P.ordering_random(g.n, 1)
    return g, o, port.factor(g, o.perm, 3)


@pytest.mark.parametrize("defect", ["row_on_diagonal", "row_above", "row_out_of_range", "col_ptr_decreasing",
                                    "col_ptr_nonzero_start", "perm_repeat"])
def test_malformed_factor_rejected(gpu_ctx, port, defect):
    g, o, want = _good(port)
    f = factor_from_port(want)
    col_ptr, rows, perm = f.col_ptr.copy(), f.rows.copy(), f.perm.copy()
    k = int(np.argmax(np.diff(col_ptr) > 0))  # a column with entries
    if defect == "row_on_diagonal":
        rows[col_ptr[k]] = k
    elif defect == "row_above":
        rows[col_ptr[k + 1] - 1] = max(k - 1, 0)
    elif defect == "row_out_of_range":
        rows[col_ptr[k]] = f.n + 5
    elif defect == "col_ptr_decreasing":
        col_ptr[k + 1] = col_ptr[k] - 1
    elif defect == "col_ptr_nonzero_start":
        col_ptr[0] = 1
    else:
        perm[1] = perm[0]
    bad = P.LdlFactor(f.n, col_ptr, rows, f.values, f.diag, perm)
    r = P.make_rhs(g, "random_projected", 0)
    with pytest.raises(P.Error) as ei:
        P.apply_preconditioner_gpu(bad, r, ctx=gpu_ctx)
    want_code = P.Errc.not_a_permutation if defect == "perm_repeat" else P.Errc.dimension_mismatch
    assert ei.value.code == want_code
    # the context still works, and nothing of the rejected factor is resident
    z = P.apply_preconditioner_gpu(f, r, ctx=gpu_ctx)
    assert z.tobytes() == port.apply_preconditioner(want, r).tobytes()


def test_batch_member_perm_checked(gpu_ctx):
    # problem 0 perm [0, 2] and problem 1 perm [-1] form a valid union [0, 2, 1]
    g0 = P.LaplacianGraph.from_edges(2, [(0, 1, 1.0)])
    g1 = P.LaplacianGraph.from_edges(1, [])
    import ctypes as C
    from paper_2505_02977_b200 import _lib as L
    lib = P.rchol.lib
    csrs = (L.parac_csr * 2)(g0.csr(), g1.csr())
    p0 = np.array([0, 2], np.int32)
    p1 = np.array([-1], np.int32)
    perms = (C.c_void_p * 2)(p0.ctypes.data, p1.ctypes.data)
    seeds = np.zeros(2, np.uint64)
    rc = lib.parac_gpu_upload_batch(gpu_ctx.handle, 2, csrs, perms, seeds.ctypes.data)
    assert rc == P.Errc.not_a_permutation
    assert b"batch problem 0" in lib.parac_gpu_last_error()
    # the failed staging left nothing resident
    assert lib.parac_gpu_factor_resident(gpu_ctx.handle, 0, None, None) == P.Errc.dimension_mismatch
    gpu_ctx._graph = None
    gpu_ctx._resident = None


def test_failed_factor_drops_resident_state(gpu_ctx, port):
    # an attempt that fails (caller budget too small -> ArenaExhausted) must not
    # leave the previous factor marked resident over its reused buffers
    g, o, want = _good(port)
    f = P.factor_gpu(g, o, 3, ctx=gpu_ctx)
    assert f.same_values(factor_from_port(want))
    with pytest.raises(P.Error) as ei:
        P.factor_gpu(g, o, 3, P.GpuOptions(fill_pool_entries=1, column_arena_entries=1, first_chunk=1), ctx=gpu_ctx)
    assert ei.value.code == P.Errc.arena_exhausted
    import ctypes as C
    lib = P.rchol.lib
    col_ptr = np.empty(g.n + 1, np.int64)
    assert lib.parac_gpu_download(gpu_ctx.handle, col_ptr.ctypes.data, None, None, None, None, None,
                                  None) == P.Errc.dimension_mismatch
    gpu_ctx._resident = None
