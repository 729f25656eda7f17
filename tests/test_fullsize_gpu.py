"""GPU parity at the BASELINE.json configuration sizes, against reference
output computed by the unmodified reference (tests/golden/fullsize.json, made
by tests/golden/make_fullsize.py from oracle/_ref):

  * factor checksum (LdlFactor::checksum, src/factor.cpp:17-36), nnz, total
    fills and the FactorStats digest -- bit-exact, as at small sizes;
  * PCG to 1e-8 on the GPU factor: iterations within 10% of the reference's
    pcg_solve on the reference factor (north_star), true relative residual <= tol;
  * the batch configuration's 64 problems (64^3, ordering_random(n, i), seed i).

R-MAT scale 22 (64M edges) runs by default (~23 s on one B200, mostly host-side
graph generation; PARAC_SKIP_FULLSIZE_RMAT=1 skips it); its reference checksum
is pinned in the fixture.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2505_02977_b200 as P

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(ROOT, "tests", "golden", "fullsize.json")) as fh:
    FULL = json.load(fh)
CFG = {c["name"]: c for c in FULL["configs"]}

BUILDERS = {
    "poisson2d_256": lambda: P.gen_poisson2d(256),
    "poisson3d_128": lambda: P.gen_poisson3d(128),
    "poisson27_96": lambda: P.gen_poisson27(96, 1),
    "rmat_22": lambda: P.gen_rmat(22, 16, 0),
}


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def run_config(ctx, name):
    e = CFG[name]
    g = BUILDERS[name]()
    assert digest(g.ptr, g.adj, g.w) == e["graph_digest"], "host generator drifted from the fixture"
    o = P.ordering_random(g.n, e["seed"])
    assert digest(o.perm) == e["perm_digest"]
    st = P.FactorStats()
    f = P.factor_gpu(g, o, e["seed"], P.GpuOptions(), st, ctx=ctx)
    assert f"{f.checksum():016x}" == e["checksum"], name
    assert f.nnz_off_diagonal() == e["nnz_off"]
    assert st.total_fills == e["total_fills"]
    assert digest(st.merged_degree, st.samples_emitted, st.fills_received) == e["stats_digest"]
    return g, f, e


@pytest.mark.parametrize("name", ["poisson2d_256", "poisson3d_128", "poisson27_96"])
def test_fullsize_factor_and_pcg(gpu_ctx, name):
    g, f, e = run_config(gpu_ctx, name)
    want = e["pcg"]
    b = P.make_rhs(g, "random_projected", 0)
    x, rep = P.rchol._pcg_resident(gpu_ctx, b, P.SolveConfig(tol=want["tol"]))
    assert rep.converged and rep.relative_residual <= want["tol"]
    it = want["iterations"]
    assert abs(rep.iterations - it) <= max(1, it // 10), (rep.iterations, it)
    assert np.isfinite(x).all() and abs(x.mean()) < 1e-9 * (np.abs(x).max() + 1)


@pytest.mark.skipif(os.environ.get("PARAC_SKIP_FULLSIZE_RMAT") == "1", reason="PARAC_SKIP_FULLSIZE_RMAT=1")
def test_fullsize_rmat22(gpu_ctx):
    # ~23 s on one B200 (host R-MAT generation + an 8.4 s factorization)
    run_config(gpu_ctx, "rmat_22")


def test_batch_64x64_checksums(gpu_ctx):
    # config[4]: all 64 problems in one device pass, each equal to the reference
    g = P.gen_poisson3d(64)
    ents = FULL["batch_64x64"]
    fs, _ = P.factor_batch_gpu([g] * len(ents), [P.ordering_random(g.n, e["i"]) for e in ents],
                               [e["i"] for e in ents], ctx=gpu_ctx)
    for e, f in zip(ents, fs):
        assert f"{f.checksum():016x}" == e["checksum"], e["i"]
        assert f.nnz_off_diagonal() == e["nnz_off"]
    # and one of them stand-alone
    f0 = P.factor_gpu(g, P.ordering_random(g.n, 5), 5, ctx=gpu_ctx)
    assert f"{f0.checksum():016x}" == ents[5]["checksum"]
