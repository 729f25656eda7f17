"""Device ordering_nnz_sort (reference proj/src/ordering.cpp:49-70)
against the host restatement (itself pinned to the reference's own outputs by
tests/test_host.py golden vectors), on graphs that take both device paths:
packed 64-bit keys (max degree < 2^11) and the two-pass sort (R-MAT hubs).
End to end: 128^3 with the device nnz-sort ordering factors to the reference
checksum the survey captured from the unmodified reference.
"""
import numpy as np
import pytest

import paper_2505_02977_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,build,seed", [
    ("poisson3d_24", lambda: P.gen_poisson3d(24), 0),
    ("poisson27_20", lambda: P.gen_poisson27(20, 1), 3),
    ("poisson2d_64", lambda: P.gen_poisson2d(64), 11),
    ("random_connected", lambda: P.gen_random_connected(5000, 20000, 7, False), 5),
    ("rmat_16", lambda: P.gen_rmat(16, 16, 0), 0),  # max degree > 2^11: two-pass path
    # many radix tiles with a ragged last tile (4096-element tiles), both paths
    ("random_connected_ragged", lambda: P.gen_random_connected(100_003, 300_000, 2, False), 1),
    ("rmat_18", lambda: P.gen_rmat(18, 8, 1), 2),
])
def test_nnz_sort_device_equals_host(gpu_ctx, name, build, seed):
    g = build()
    want = P.ordering_nnz_sort(g, seed).perm
    got = P.ordering_nnz_sort_gpu(g, seed, ctx=gpu_ctx).perm
    assert np.array_equal(got, want), name
    assert np.array_equal(np.sort(got), np.arange(g.n))


def test_nnz_sort_device_tiny(gpu_ctx):
    for n in (1, 2, 3):
        g = P.gen_random_connected(n, 0, 1, True)
        assert np.array_equal(P.ordering_nnz_sort_gpu(g, 9, ctx=gpu_ctx).perm, P.ordering_nnz_sort(g, 9).perm)


def test_nnz_sort_128_known_checksum(gpu_ctx):
    g = P.gen_poisson3d(128)
    o = P.ordering_nnz_sort_gpu(g, 0, ctx=gpu_ctx)
    f = P.factor_gpu(g, o, 0, ctx=gpu_ctx)
    assert f"{f.checksum():016x}" == "0eeae3519f0e7093"
