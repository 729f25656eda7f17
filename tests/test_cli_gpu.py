"""`parac`-compatible runner with the gpu backend, checked
against the UNMODIFIED reference (oracle/_ref) on the same graph, ordering and
seed: factor files byte-identical to the reference's write_factor of its own
factor, stats / --trace JSON equal to the reference's FactorStats and
schedule_levels, bench rows in the parac-bench-v1 schema with the reference's
checksums and PCG iteration counts within 10%.
"""
import csv
import json

import numpy as np
import pytest

import oracle
from oracle import C
import paper_2505_02977_b200 as P
from paper_2505_02977_b200 import cli

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.Reference.available(), reason="oracle/_ref not built")]


@pytest.fixture(scope="module")
def R():
    return oracle.Reference()


def ref_pcg_iters(R, h, f, seed, tol):
    n = R.L.pref_graph_n(h)
    b = np.empty(n)
    R._chk(R.L.pref_make_rhs(h, 1, seed, b.ctypes.data))
    x = np.empty(n)
    it, conv = C.c_int(), C.c_int()
    rel, rec, sec = C.c_double(), C.c_double(), C.c_double()
    R._chk(R.L.pref_pcg(h, f, b.ctypes.data, tol, 1000, x.ctypes.data, C.byref(it), C.byref(rel), C.byref(rec),
                        C.byref(conv), C.byref(sec)))
    return it.value


def test_factor_command(R, tmp_path):
    g = P.gen_poisson3d(12, "contrast", 1e-3, 1e4, 0)
    seed = 3
    stem, sj, tj = str(tmp_path / "f"), str(tmp_path / "s.json"), str(tmp_path / "t.json")
    rc = cli.main(["factor", "--gen", "poisson3d:n=12,variant=contrast", "--ordering", "random", "--seed", str(seed),
                   "--output", stem, "--stats", sj, "--trace", tj])
    assert rc == 0
    h = R.graph_from_csr(g)
    perm = P.ordering_random(g.n, seed).perm
    f, _ = R.factor(h, perm, seed, backend=R.LEFT, workers=2, stats=True)
    R._chk(R.L.pref_write_factor(f, str(tmp_path / "ref").encode()))
    for ext in (".G.mtx", ".D.mtx"):
        assert open(stem + ext, "rb").read() == open(str(tmp_path / "ref") + ext, "rb").read(), ext
    assert [int(x) for x in open(stem + ".perm.txt")] == perm.tolist()
    st = json.load(open(sj))
    rs = R.factor_stats(f)
    assert st["checksum"] == R.checksum(f)
    assert st["nnz_g"] == R.L.pref_factor_nnz_off(f) + g.n
    assert st["schedule_depth"] == R.L.pref_schedule_depth(f)
    assert st["total_fills"] == rs["total_fills"]
    assert st["fill_ratio"] == 2.0 * st["nnz_g"] / (int(g.ptr[g.n]) + g.n)
    assert st["config"]["backend"] == "gpu" and st["config"]["seed"] == seed
    # SURVEY §5 device metrics next to the reference's keys
    assert 0 < st["device_seconds"] <= st["wall_seconds"]
    assert 0 < st["eliminate_seconds"] <= st["device_seconds"]
    assert st["hbm_gbs"] > 0 and 0 < st["roofline_fraction"] < 1
    assert st["algorithmic_bytes"] == (16 * (g.n + 1) + 8 * g.n + 12 * g.num_edges() + 40 * st["total_fills"]
                                       + 20 * (st["nnz_g"] - g.n))
    tr = json.load(open(tj))
    levels = np.empty(g.n, np.int32)
    R._chk(R.L.pref_schedule_levels(f, levels.ctypes.data))
    assert tr["rounds"] == st["schedule_depth"] and tr["n"] == g.n
    inv = np.argsort(perm)
    for k in (0, 1, g.n // 2, g.n - 1):
        v = tr["vertices"][k]
        assert v["position"] == k and v["label"] == inv[k] and v["round"] == levels[k]
        assert v["fills"] == rs["fills_received"][k] and v["samples"] == rs["samples_emitted"][k]
    R.free_factor(f)
    R.free_graph(h)


def test_solve_from_reference_factor_files(R, tmp_path):
    g = P.gen_poisson3d(14)
    h = R.graph_from_csr(g)
    perm = P.ordering_random(g.n, 0).perm
    f, _ = R.factor(h, perm, 0, backend=R.SEQ)
    stem = str(tmp_path / "ref")
    R._chk(R.L.pref_write_factor(f, stem.encode()))
    R._chk(R.L.pref_write_permutation((stem + ".perm.txt").encode(), g.n, perm.ctypes.data))
    rj, xs = str(tmp_path / "r.json"), str(tmp_path / "x.mtx")
    rc = cli.main(["solve", "--gen", "poisson3d:n=14", "--factor", stem, "--tol", "1e-8", "--report", rj,
                   "--solution", xs])
    rep = json.load(open(rj))
    assert rc == 0 and rep["converged"]
    it = ref_pcg_iters(R, h, f, 0, 1e-8)
    assert abs(rep["iterations"] - it) <= max(1, it // 10)
    assert len(P.read_vector(xs)) == g.n
    R.free_factor(f)
    R.free_graph(h)


def test_bench_rows(R, tmp_path):
    out = str(tmp_path / "b.csv")
    specs = ["poisson3d:n=10", "poisson3d:n=12,variant=anisotropic"]
    rc = cli.main(["bench", "--gens", ";".join(specs), "--orderings", "random,nnz-sort", "--seeds", "0,1",
                   "--solve", "--tol", "1e-8", "--csv", out])
    assert rc == 0
    rows = list(csv.DictReader(open(out)))
    assert len(rows) == 2 * 2 * 2
    graphs = {specs[0]: P.gen_poisson3d(10), specs[1]: P.gen_poisson3d(12, "anisotropic", 1e-3, 1e4, 0)}
    for r in rows:
        assert r["schema"] == "parac-bench-v1" and r["error"] == "" and r["backend"] == "gpu"
        g = graphs[r["input"]]
        seed = int(r["seed"])
        h = R.graph_from_csr(g)
        perm = P.ordering_random(g.n, seed).perm if r["ordering"] == "random" else R.ordering_nnz_sort(h, seed)
        f, _ = R.factor(h, perm, seed, backend=R.SEQ)
        assert int(r["checksum"]) == R.checksum(f), r
        assert int(r["nnz_g"]) == R.L.pref_factor_nnz_off(f) + g.n
        assert int(r["schedule_depth"]) == R.L.pref_schedule_depth(f)
        it = ref_pcg_iters(R, h, f, seed, 1e-8)
        assert r["converged"] == "1" and abs(int(r["iterations"]) - it) <= max(1, it // 10), (r, it)
        assert float(r["speedup_vs_w1"]) == 1.0
        R.free_factor(f)
        R.free_graph(h)


def test_cli_errors():
    assert cli.main(["factor", "--gen", "poisson3d:n=4", "--backend", "par-left"]) == 10 + 5
    assert cli.main(["factor", "--gen", "poisson3d:n=4", "--ordering", "bogus"]) == 10 + 5
    assert cli.main(["factor", "--gen", "cube:n=4"]) == 10 + 5
    assert cli.main(["factor", "--input", "/nonexistent.mtx"]) == 10 + 16


def test_solve_factors_on_gpu_without_factor_files(R, tmp_path):
    # solve without --factor: the runner factors on the device (gpu backend), then runs PCG
    g = P.gen_poisson3d(12, "anisotropic", 1e-3, 1e4, 0)
    rj = str(tmp_path / "r.json")
    rc = cli.main(["solve", "--gen", "poisson3d:n=12,variant=anisotropic", "--ordering", "random", "--seed", "2",
                   "--tol", "1e-8", "--report", rj])
    rep = json.load(open(rj))
    assert rc == 0 and rep["converged"] and rep["relative_residual"] <= 1e-8
    h = R.graph_from_csr(g)
    f, _ = R.factor(h, P.ordering_random(g.n, 2).perm, 2, backend=R.SEQ)
    it = ref_pcg_iters(R, h, f, 2, 1e-8)
    assert abs(rep["iterations"] - it) <= max(1, it // 10)
    R.free_factor(f)
    R.free_graph(h)
