"""GPU: the sm_100a factorization is byte-identical (LdlFactor::same_values,
proj/src/factor.cpp:10-13) to the oracle on the reference's test corpus, and
its FactorStats agree (proj/tests/test_factor_par.cpp:172-190)."""
import numpy as np
import pytest

import paper_2505_02977_b200 as P
from corpus import case, digest, factor_from_port

pytestmark = pytest.mark.gpu


def gpu_factor(ctx, g, perm, seed, **opts):
    stats = P.FactorStats()
    f = P.factor_gpu(g, P.Ordering(perm), seed, P.GpuOptions(**opts), stats, ctx=ctx)
    return f, stats


def assert_same(f, ref_f, name=""):
    assert f.same_values(ref_f), name


def test_golden_corpus_byte_identical(gpu_ctx, port, gold):
    for e in gold["factors"]:
        g, perm, seed = case(e["name"])
        f, st = gpu_factor(gpu_ctx, g, perm, seed, verify=True)
        assert f"{f.checksum():016x}" == e["checksum"], e["name"]
        want = port.factor(g, perm, seed)
        assert_same(f, factor_from_port(want), e["name"])
        assert np.array_equal(st.merged_degree, want["merged_degree"]), e["name"]
        assert np.array_equal(st.samples_emitted, want["samples_emitted"]), e["name"]
        assert np.array_equal(st.fills_received, want["fills_received"]), e["name"]
        assert st.total_fills == e["total_fills"]


@pytest.mark.parametrize("opts", [dict(grid_ctas=1), dict(first_chunk=1), dict(first_chunk=2, grid_ctas=3),
                                  dict(delay_ns=2000, verify=True)])
def test_schedule_and_pool_shape_do_not_change_bits(gpu_ctx, port, opts):
    # the claim order, CTA count and fill-chunk layout must never move a bit
    for name in ("poisson16_random0", "rc200_s1_nnz", "components3000_s0"):
        g, perm, seed = case(name)
        f, _ = gpu_factor(gpu_ctx, g, perm, seed, **opts)
        assert_same(f, factor_from_port(port.factor(g, perm, seed)), name)


def test_repeat_stress(gpu_ctx, port):
    # proj/tests/test_factor_par.cpp:146-170 (delay injection, 25 runs)
    g = P.gen_random_connected(200, 360, 17)
    perm = P.ordering_random(200, 3).perm
    want = factor_from_port(port.factor(g, perm, 5))
    for run in range(25):
        f, _ = gpu_factor(gpu_ctx, g, perm, 5, verify=True, delay_ns=500 * (run % 5))
        assert_same(f, want)


@pytest.mark.parametrize("builder,seed", [
    (lambda: P.gen_poisson2d(64), 0),
    (lambda: P.gen_poisson27(12, 1), 0),
    (lambda: P.gen_poisson3d(24, "contrast", contrast_ratio=1e6, seed=1), 3),
    (lambda: P.gen_rmat(12, 16, 0), 0),
    (lambda: P.gen_random_components(5000, 7, 20000, 2), 4),
])
def test_paper_shapes_byte_identical(gpu_ctx, port, builder, seed):
    g = builder()
    for perm in (P.ordering_random(g.n, seed).perm, P.ordering_nnz_sort(g, seed).perm):
        f, st = gpu_factor(gpu_ctx, g, perm, seed)
        want = port.factor(g, perm, seed)
        assert_same(f, factor_from_port(want))
        assert np.array_equal(st.fills_received, want["fills_received"])


def test_poisson64_matches_reference_checksum(gpu_ctx, gold):
    e = next(x for x in gold["factors"] if x["name"] == "poisson64_random0")
    g, perm, seed = case(e["name"])
    f, _ = gpu_factor(gpu_ctx, g, perm, seed)
    assert f"{f.checksum():016x}" == e["checksum"] == "3bbec4ec5f0cad7b"


def test_edge_cases(gpu_ctx, port):
    # empty graph, isolated vertices, single vertex, two vertices
    for n, edges in ((1, []), (6, []), (2, [(0, 1, 2.5)]), (5, [(1, 3, 1.0)])):
        g = P.LaplacianGraph.from_edges(n, edges)
        for s in range(3):
            perm = P.ordering_random(n, s).perm
            f, _ = gpu_factor(gpu_ctx, g, perm, s)
            assert_same(f, factor_from_port(port.factor(g, perm, s)))


def test_arena_exhaustion_is_clean(gpu_ctx):
    # proj/tests/test_factor_par.cpp:105-118: explicit tiny budgets fail cleanly
    g = P.gen_random_connected(100, 300, 3)
    perm = P.ordering_random(100, 1).perm
    with pytest.raises(P.Error) as ei:
        gpu_factor(gpu_ctx, g, perm, 0, column_arena_entries=64)
    assert ei.value.code == P.Errc.arena_exhausted
    with pytest.raises(P.Error) as ei:
        gpu_factor(gpu_ctx, g, perm, 0, fill_pool_entries=4, first_chunk=1)
    assert ei.value.code == P.Errc.arena_exhausted
    # the context stays usable afterwards
    f, _ = gpu_factor(gpu_ctx, g, perm, 0)
    assert f.nnz_off_diagonal() > 0


def test_dimension_mismatch(gpu_ctx):
    g = P.gen_poisson3d(4)
    with pytest.raises(P.Error) as ei:
        P.factor_gpu(g, P.Ordering.identity(10), 0, ctx=gpu_ctx)
    assert ei.value.code == P.Errc.dimension_mismatch


def test_native_library_is_what_ran(gpu_ctx):
    before = P.rchol.lib.parac_gpu_launch_count()
    g, perm, seed = case("poisson16_random0")
    gpu_factor(gpu_ctx, g, perm, seed)
    assert P.rchol.lib.parac_gpu_launch_count() > before


def test_batch_union_equals_standalone(gpu_ctx, port, gold):
    # config[4] mechanism: several independent problems factored in one device
    # pass (disjoint union, per-problem seeds/keys) -- each factor byte-identical
    # to the reference's stand-alone factorization, whatever its size and seed
    names = ["p3", "k3_s7", "star8", "rc200_s1_nnz", "poisson16_random1", "components3000_s2", "ring9_s3"]
    cases = [case(nm) for nm in names]
    fs, info = P.factor_batch_gpu([c[0] for c in cases], [P.Ordering(c[1]) for c in cases],
                                  [c[2] for c in cases], ctx=gpu_ctx)
    for nm, (g, perm, seed), f in zip(names, cases, fs):
        assert_same(f, factor_from_port(port.factor(g, perm, seed)), nm)
        e = next(x for x in gold["factors"] if x["name"] == nm)
        assert f"{f.checksum():016x}" == e["checksum"], nm


def test_batch_with_hub_members(gpu_ctx, port):
    """Hub columns inside a batch: R-MAT members (several hub jobs at once,
    per-member sample keys inside the cooperative phases) next to a mesh,
    each member byte-identical to its stand-alone factorization."""
    gs = [P.gen_rmat(13, 16, 1), P.gen_poisson3d(12), P.gen_rmat(12, 16, 2)]
    perms = [P.ordering_random(g.n, i).perm for i, g in enumerate(gs)]
    seeds = [5, 6, 7]
    fs, info = P.factor_batch_gpu(gs, [P.Ordering(p) for p in perms], seeds, ctx=gpu_ctx)
    assert info.large_columns > 0, "no member column took the hub path"
    for i, (g, perm, seed, f) in enumerate(zip(gs, perms, seeds, fs)):
        assert_same(f, factor_from_port(port.factor(g, perm, seed)), f"member {i}")


@pytest.mark.parametrize("scale,opts", [(15, {}), (16, {}), (15, dict(grid_ctas=2)),
                                        (15, dict(grid_ctas=9, verify=True)),
                                        (15, dict(delay_ns=3000, verify=True))])
def test_rmat_wide_columns_byte_identical(gpu_ctx, port, scale, opts):
    # R-MAT hubs exceed the shared-memory column capacity (1024 raw entries):
    # the cooperative hub path (phases in 256-entry chunks taken by waiting
    # big CTAs; with grid_ctas=2 the owner works alone) -- still byte-identical
    # to the reference restatement, whoever takes which chunk
    g = P.gen_rmat(scale, 16, 0)
    perm = P.ordering_random(g.n, 0).perm
    f, st = gpu_factor(gpu_ctx, g, perm, 0, **opts)
    assert st.large_columns > 0, "no column took the wide path"
    want = port.factor(g, perm, 0)
    assert_same(f, factor_from_port(want))
    assert np.array_equal(st.fills_received, want["fills_received"])


@pytest.mark.parametrize("grid", [0, 2, 7])
def test_star_center_first_dependency_trace(gpu_ctx, port, grid):
    """proj/tests/test_factor_par.cpp:67-103 on the device: TestHooks::on_phase's
    dp snapshots while position 0 (the star's centre) is eliminated. The seed's
    first draw pairs leaves 1 and 2, so the samples are {(1,2), (2,3)} and the
    counters go (0,1,1,1) -> (0,1,2,2) after the samples -> (0,0,1,1) after the
    decrements; the factor is the full chain rows {1,2,3,2,3}."""
    from corpus import star
    salt = 0x73616D706C696E67  # kSaltSampling ("sampling"), proj/include/parac/rng.hpp
    chosen = next(s for s in range(64) if port.unit_uniform(port.derive_seed(s, salt), 0, 0) * 2.0 >= 1.0)
    g = star(3)
    f, _ = gpu_factor(gpu_ctx, g, np.arange(4, dtype=np.int32), chosen, trace_position=0, grid_ctas=grid)
    snaps = gpu_ctx.phase_snapshots()
    assert set(snaps) == {"gathered", "sampled", "decremented"}
    assert snaps["gathered"].tolist() == [0, 1, 1, 1]
    assert snaps["sampled"].tolist() == [0, 1, 2, 2]
    assert snaps["decremented"].tolist() == [0, 0, 1, 1]
    assert f.rows.tolist() == [1, 2, 3, 2, 3]
    # a later run without tracing: no snapshots, same factor
    f2, _ = gpu_factor(gpu_ctx, g, np.arange(4, dtype=np.int32), chosen)
    assert f2.same_values(f)
    with pytest.raises(P.Error):
        gpu_ctx.phase_snapshots()


def test_phase_trace_on_a_cta_column(gpu_ctx, port):
    """The CTA path (raw column > 128 entries) takes the same snapshots: the
    hub of a 300-leaf star, eliminated first. Its rows are published only
    after the "decremented" snapshot, so nothing else runs in between."""
    from corpus import star
    g = star(300)
    perm = np.arange(301, dtype=np.int32)
    f, st = gpu_factor(gpu_ctx, g, perm, 1, trace_position=0)
    want = port.factor(g, perm, 1)
    assert f.same_values(P.LdlFactor(want["n"], want["col_ptr"], want["rows"], want["values"], want["diag"],
                                     want["perm"]))
    snaps = gpu_ctx.phase_snapshots()
    dp0 = P.dependency_counts(g, P.Ordering.identity(301))
    assert snaps["gathered"].tolist() == dp0.tolist()
    # every emitted fill raised its hi endpoint's counter by one
    assert int((snaps["sampled"] - snaps["gathered"]).sum()) == int(st.samples_emitted[0]) > 0
    assert (snaps["sampled"] >= snaps["gathered"]).all()
    # the hub's decrements: one per leaf (multiplicity 1)
    assert snaps["decremented"][0] == 0
    assert (snaps["decremented"][1:] == snaps["sampled"][1:] - 1).all()


def test_phase_trace_on_a_hub_column(gpu_ctx, port):
    """The cooperative hub path (raw column > 1024 entries) takes the
    snapshots at the same phase boundaries: the centre of a 1500-leaf star,
    eliminated first while every leaf waits on it."""
    from corpus import star
    g = star(1500)
    perm = np.arange(1501, dtype=np.int32)
    f, st = gpu_factor(gpu_ctx, g, perm, 2, trace_position=0, verify=True)
    assert st.large_columns > 0, "the centre did not take the hub path"
    want = port.factor(g, perm, 2)
    assert f.same_values(P.LdlFactor(want["n"], want["col_ptr"], want["rows"], want["values"], want["diag"],
                                     want["perm"]))
    snaps = gpu_ctx.phase_snapshots()
    dp0 = P.dependency_counts(g, P.Ordering.identity(1501))
    assert snaps["gathered"].tolist() == dp0.tolist()
    assert int((snaps["sampled"] - snaps["gathered"]).sum()) == int(st.samples_emitted[0]) > 0
    assert (snaps["sampled"] >= snaps["gathered"]).all()
    # the centre's own counter is zero (leaves made ready are published by the
    # chunks that decremented them, so later eliminations may already have
    # moved the leaves' counters by the time of this snapshot)
    assert snaps["decremented"][0] == 0


def test_hub_column_on_the_mesh_kernel_instance_reruns(gpu_ctx, port, monkeypatch):
    """A column wider than 1024 raw entries met by the kernel instance without
    the hub path (chosen for graphs without hub vertices; forced here) aborts
    the pass, and the library re-runs it with the hub path: same bits."""
    monkeypatch.setenv("PARAC_HUBS", "0")
    g = P.gen_rmat(12, 16, 0)
    perm = P.ordering_random(g.n, 0).perm
    f, st = gpu_factor(gpu_ctx, g, perm, 0)
    assert st.large_columns > 0 and st.attempts == 2
    assert f.same_values(factor_from_port(port.factor(g, perm, 0)))
    # without the override the instance with the hub path runs first
    monkeypatch.delenv("PARAC_HUBS")
    f2, st2 = gpu_factor(gpu_ctx, g, perm, 0)
    assert st2.attempts == 1 and f2.same_values(f)
