"""GPU: the streamed assembly and download (parac_gpu_factor_begin / _end,
stream_assemble.cu). The CSC factor is assembled beside the elimination and
copied to the host while it runs; the result must be the bytes of the
after-the-fact assembly (launch_assemble) and of the oracle
(LdlFactor::same_values, proj/src/factor.cpp:10-13), whatever the output
memory (pinned or pageable), the schedule, or a re-run of the pass."""
import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import case, factor_from_port

pytestmark = pytest.mark.gpu


def streamed(ctx, g, perm, seed, out=None, capacity=None, **opts):
    ctx.upload(g, P.Ordering(perm))
    info, (cp, rows, vals, diag) = ctx.factor_to_host(seed, P.GpuOptions(**opts), out=out, capacity=capacity)
    z = info.nnz_off_diagonal
    return P.LdlFactor(g.n, cp.copy(), rows[:z].copy(), vals[:z].copy(), diag[:g.n].copy(), perm), info


def after_the_fact(ctx, g, perm, seed, monkeypatch, **opts):
    monkeypatch.setenv("PARAC_STREAM", "0")
    f = P.factor_gpu(g, P.Ordering(perm), seed, P.GpuOptions(**opts), ctx=ctx)
    monkeypatch.delenv("PARAC_STREAM")
    return f


@pytest.mark.parametrize("builder,seed", [
    (lambda: P.gen_poisson3d(24), 0),          # 7 blocks of 2048 positions
    (lambda: P.gen_poisson2d(100), 1),         # 5 blocks, the last one partial
    (lambda: P.gen_poisson27(10, 1), 0),       # one partial block
    (lambda: P.gen_rmat(13, 16, 0), 0),        # hub columns (cooperative path)
    (lambda: P.gen_random_components(3000, 4, 9000, 2), 2),  # components, m == 0 columns
])
def test_streamed_factor_is_the_assembled_factor(gpu_ctx, port, monkeypatch, builder, seed):
    g = builder()
    perm = P.ordering_random(g.n, seed).perm
    want = factor_from_port(port.factor(g, perm, seed))
    base = after_the_fact(gpu_ctx, g, perm, seed, monkeypatch)
    assert base.same_values(want)
    cap = want.nnz_off_diagonal()
    f, info = streamed(gpu_ctx, g, perm, seed, capacity=cap)
    assert info.attempts >= 1 and info.nnz_off_diagonal == cap
    assert f.same_values(want)
    # the resident copy the streamer assembled is what solves and downloads see
    f2, _ = gpu_ctx.download(with_stats=False)
    assert f2.same_values(want)


def test_pinned_outputs(gpu_ctx, port):
    torch = pytest.importorskip("torch")
    g = P.gen_poisson3d(20)
    perm = P.ordering_random(g.n, 4).perm
    want = factor_from_port(port.factor(g, perm, 4))
    z = want.nnz_off_diagonal()
    bufs = [torch.empty(k, dtype=dt, pin_memory=True).numpy()
            for k, dt in ((g.n + 1, torch.int64), (z, torch.int32), (z, torch.float64), (g.n, torch.float64))]
    for a in bufs:
        a.fill(0)
    f, _ = streamed(gpu_ctx, g, perm, 4, out=tuple(bufs))
    assert f.same_values(want)


@pytest.mark.parametrize("opts", [dict(grid_ctas=2), dict(grid_ctas=5, first_chunk=1),
                                  dict(delay_ns=3000, verify=True)])
def test_streamed_under_other_schedules(gpu_ctx, port, opts):
    g, perm, seed = case("poisson16_random0")
    want = factor_from_port(port.factor(g, perm, seed))
    f, _ = streamed(gpu_ctx, g, perm, seed, capacity=want.nnz_off_diagonal(), **opts)
    assert f.same_values(want)


def test_rerun_with_the_hub_path_restreams(gpu_ctx, port, monkeypatch):
    # the mesh instance aborts on the first wide column; the second pass
    # streams everything again over the first pass's partial output
    monkeypatch.setenv("PARAC_HUBS", "0")
    g = P.gen_rmat(12, 16, 0)
    perm = P.ordering_random(g.n, 0).perm
    want = factor_from_port(port.factor(g, perm, 0))
    out = (np.full(g.n + 1, -7, np.int64), np.full(want.nnz_off_diagonal(), -7, np.int32),
           np.full(want.nnz_off_diagonal(), np.nan), np.full(g.n, np.nan))
    f, info = streamed(gpu_ctx, g, perm, 0, out=out)
    assert info.attempts == 2
    assert f.same_values(want)


def test_capacity_too_small_keeps_the_factor_resident(gpu_ctx, port):
    g = P.gen_poisson3d(16)
    perm = P.ordering_random(g.n, 2).perm
    want = factor_from_port(port.factor(g, perm, 2))
    z = want.nnz_off_diagonal()
    gpu_ctx.upload(g, P.Ordering(perm))
    with pytest.raises(P.Error) as ei:
        gpu_ctx.factor_to_host(2, capacity=z // 3)
    assert ei.value.code == P.Errc.budget_exceeded
    f, _ = gpu_ctx.download(with_stats=False)
    assert f.same_values(want)


def test_begin_end_protocol_errors(gpu_ctx):
    lib = P.rchol.lib
    L = P.rchol.L
    info = L.parac_gpu_factor_info()
    # end without begin
    rc = lib.parac_gpu_factor_end(gpu_ctx.handle, info, None, None, None, None, 0)
    assert rc == P.Errc.internal_error
    g = P.gen_poisson3d(8)
    gpu_ctx.upload(g, P.ordering_random(g.n, 0))
    o = P.GpuOptions().native()
    assert lib.parac_gpu_factor_begin(gpu_ctx.handle, 0, o) == 0
    # a second begin while one is pending
    assert lib.parac_gpu_factor_begin(gpu_ctx.handle, 0, o) == P.Errc.internal_error
    # nothing else touches the context's buffers while it is pending
    assert lib.parac_gpu_upload(gpu_ctx.handle, g.csr(), P.ordering_random(g.n, 0).perm.ctypes.data) == \
        P.Errc.internal_error
    assert lib.parac_gpu_factor_end(gpu_ctx.handle, info, None, None, None, None, 0) == 0
    assert info.n == g.n and info.nnz_off_diagonal > 0
    # explicit budgets fail cleanly through _end, and the context recovers
    o.column_arena_entries = 64
    assert lib.parac_gpu_factor_begin(gpu_ctx.handle, 0, o) == 0
    assert lib.parac_gpu_factor_end(gpu_ctx.handle, info, None, None, None, None, 0) == P.Errc.arena_exhausted
    f = P.factor_gpu(g, P.ordering_random(g.n, 0), 0, ctx=gpu_ctx)
    assert f.nnz_off_diagonal() > 0


def batch_members():
    gs = [P.gen_poisson3d(20), P.gen_random_connected(300, 500, 3), P.gen_rmat(12, 16, 1),
          P.gen_poisson2d(70), P.gen_random_connected(5, 4, 1)]
    perms = [P.ordering_random(g.n, i + 1).perm for i, g in enumerate(gs)]
    seeds = [3, 4, 5, 6, 7]
    return gs, perms, seeds


@pytest.mark.parametrize("stream", ["1", "0"])
def test_batch_streamed_members_are_standalone_factors(gpu_ctx, port, monkeypatch, stream):
    # members of 8000, 300, 4096, 4900 and 5 positions: blocks never straddle
    # members, while K3's 2048-position counters do; each member assembled
    # into its own region (or, PARAC_STREAM=0, the union CSC after K3)
    monkeypatch.setenv("PARAC_STREAM", stream)
    gs, perms, seeds = batch_members()
    fs, info = P.factor_batch_gpu(gs, [P.Ordering(p) for p in perms], seeds, ctx=gpu_ctx)
    for i, (g, perm, seed, f) in enumerate(zip(gs, perms, seeds, fs)):
        assert f.same_values(factor_from_port(port.factor(g, perm, seed))), f"member {i}"


@pytest.mark.parametrize("stream", ["1", "0"])
def test_batch_to_host_pinned_and_short_capacity(gpu_ctx, port, monkeypatch, stream):
    monkeypatch.setenv("PARAC_STREAM_BATCH", stream)
    torch = pytest.importorskip("torch")
    import ctypes as C
    lib, L = P.rchol.lib, P.rchol.L
    gs, perms, seeds = batch_members()
    want = [factor_from_port(port.factor(g, p, s)) for g, p, s in zip(gs, perms, seeds)]
    zs = [w.nnz_off_diagonal() for w in want]
    caps = np.array(zs, np.int64)
    caps[2] -= 1  # member 2's rows/values one entry short
    pin = lambda k, dt: torch.zeros(max(k, 1), dtype=dt, pin_memory=True).numpy()
    bufs = [(pin(g.n + 1, torch.int64), pin(z, torch.int32), pin(z, torch.float64), pin(g.n, torch.float64))
            for g, z in zip(gs, zs)]
    arr = [(C.c_void_p * len(gs))(*[b[j].ctypes.data for b in bufs]) for j in range(4)]
    csrs = (L.parac_csr * len(gs))(*[g.csr() for g in gs])
    pp = (C.c_void_p * len(gs))(*[p.ctypes.data for p in perms])
    sd = np.array(seeds, np.uint64)
    info = L.parac_gpu_factor_info()
    rc = lib.parac_gpu_factor_batch_to_host(gpu_ctx.handle, len(gs), csrs, pp, sd.ctypes.data,
                                            P.GpuOptions().native(), info, *arr, caps.ctypes.data)
    assert rc == P.Errc.budget_exceeded
    for i, (g, w, b) in enumerate(zip(gs, want, bufs)):
        if i == 2:
            continue
        f = P.LdlFactor(g.n, b[0], b[1][:zs[i]], b[2][:zs[i]], b[3][:g.n], perms[i])
        assert f.same_values(w), f"member {i}"
    # the short member from the resident union
    z = C.c_int64()
    assert lib.parac_gpu_batch_nnz(gpu_ctx.handle, 2, C.byref(z)) == 0 and z.value == zs[2]
    cp, r, v, d = (np.empty(gs[2].n + 1, np.int64), np.empty(zs[2], np.int32), np.empty(zs[2]),
                   np.empty(gs[2].n))
    assert lib.parac_gpu_download_batch(gpu_ctx.handle, 2, cp.ctypes.data, r.ctypes.data, v.ctypes.data,
                                        d.ctypes.data) == 0
    assert P.LdlFactor(gs[2].n, cp, r, v, d, perms[2]).same_values(want[2])


def test_batch_region_overflow_falls_back_to_the_union(gpu_ctx, port):
    # tiny explicit arena: member regions (shares of it) overflow, the library
    # assembles the union CSC after K3 instead -- or the budget fails cleanly
    gs, perms, seeds = batch_members()
    want = [factor_from_port(port.factor(g, p, s)) for g, p, s in zip(gs, perms, seeds)]
    z = sum(w.nnz_off_diagonal() for w in want)
    try:
        fs, info = P.factor_batch_gpu(gs, [P.Ordering(p) for p in perms], seeds,
                                      P.GpuOptions(column_arena_entries=z + 64, fill_pool_entries=1 << 22), ctx=gpu_ctx)
    except P.Error as e:
        assert e.code == P.Errc.arena_exhausted
        return
    for i, (f, w) in enumerate(zip(fs, want)):
        assert f.same_values(w), f"member {i}"


def test_single_and_batch_end_reject_the_other_layout(gpu_ctx):
    lib, L = P.rchol.lib, P.rchol.L
    info = L.parac_gpu_factor_info()
    g = P.gen_poisson3d(6)
    gpu_ctx.upload(g, P.ordering_random(g.n, 0))
    assert lib.parac_gpu_factor_begin(gpu_ctx.handle, 0, P.GpuOptions().native()) == 0
    assert lib.parac_gpu_factor_batch_end(gpu_ctx.handle, info, None, None, None, None, None) == \
        P.Errc.dimension_mismatch
    # the pending factorization was completed: the context is usable
    f = P.factor_gpu(g, P.ordering_random(g.n, 0), 0, ctx=gpu_ctx)
    assert f.nnz_off_diagonal() > 0
