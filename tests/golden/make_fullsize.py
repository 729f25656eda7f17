"""Generate tests/golden/fullsize.json: reference checksums and PCG iteration
counts at the BASELINE.json configuration sizes, from the UNMODIFIED reference
build (oracle/_ref). Run in the dev container (minutes; R-MAT 22 dominates):

    python tests/golden/make_fullsize.py [--skip-rmat]

Graphs come from this repo's host builders (the harness generators of SURVEY
§8(d): gen_poisson3d is the reference's own generator, re-verified bit-for-bit
by tests/test_host.py; 2D / 27-point / R-MAT are harness definitions) and are
handed to the reference through LaplacianGraph::from_edges-equivalent CSR
ingestion; the reference then factors them with factor_parallel_left
(byte-identical to factor_randomized for any worker count).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2505_02977_b200 as P  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "fullsize.json")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def configs(skip_rmat: bool):
    yield "poisson2d_256", lambda: P.gen_poisson2d(256), 0, True
    yield "poisson3d_128", lambda: P.gen_poisson3d(128), 0, True
    yield "poisson27_96", lambda: P.gen_poisson27(96, 1), 0, True
    if not skip_rmat:
        yield "rmat_22", lambda: P.gen_rmat(22, 16, 0), 0, False


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--skip-rmat", action="store_true")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 8)
    a = ap.parse_args()
    R = oracle.Reference()
    out = {"_source": "oracle/_ref (unmodified reference), factor_parallel_left", "configs": [],
           "batch_64x64": []}
    if os.path.exists(OUT):
        with open(OUT) as fh:
            old = json.load(fh)
        out["configs"] = [c for c in old.get("configs", []) if a.skip_rmat and c["name"] == "rmat_22"]
    for name, build, seed, pcg in configs(a.skip_rmat):
        t = time.time()
        g = build()
        perm = P.ordering_random(g.n, seed).perm
        h = R.graph_from_csr(g)
        f, wall = R.factor(h, perm, seed, backend=R.LEFT, workers=a.workers, stats=True)
        st = R.factor_stats(f)
        e = {"name": name, "n": g.n, "edges": int(g.num_edges()), "seed": seed,
             "graph_digest": digest(g.ptr, g.adj, g.w), "perm_digest": digest(perm),
             "checksum": f"{R.checksum(f):016x}", "nnz_off": int(R.L.pref_factor_nnz_off(f)),
             "total_fills": int(st["total_fills"]),
             "stats_digest": digest(st["merged_degree"], st["samples_emitted"], st["fills_received"]),
             "depth": int(R.L.pref_schedule_depth(f)), "ref_factor_wall_s": wall}
        if pcg:
            b = np.empty(g.n, np.float64)
            R._chk(R.L.pref_make_rhs(h, 1, 0, b.ctypes.data))
            x = np.empty(g.n, np.float64)
            it, conv = oracle.C.c_int(), oracle.C.c_int()
            rel, rec, sec = oracle.f64(), oracle.f64(), oracle.f64()
            R._chk(R.L.pref_pcg(h, f, b.ctypes.data, 1e-8, 1000, x.ctypes.data, oracle.C.byref(it),
                                oracle.C.byref(rel), oracle.C.byref(rec), oracle.C.byref(conv),
                                oracle.C.byref(sec)))
            e["pcg"] = {"tol": 1e-8, "rhs": "make_rhs(random_projected, 0)", "iterations": it.value,
                        "relative_residual": rel.value, "converged": bool(conv.value),
                        "ref_solve_s": sec.value}
        R.free_factor(f)
        R.free_graph(h)
        out["configs"].append(e)
        print(name, e["checksum"], e.get("pcg", {}).get("iterations"), f"{time.time() - t:.1f}s", flush=True)
    # config[4]: 64 x gen_poisson3d(64), problem i: ordering_random(n, i), seed i
    g = P.gen_poisson3d(64)
    h = R.graph_from_csr(g)
    for i in range(64):
        perm = P.ordering_random(g.n, i).perm
        f, _ = R.factor(h, perm, i, backend=R.LEFT, workers=a.workers)
        out["batch_64x64"].append({"i": i, "checksum": f"{R.checksum(f):016x}",
                                   "nnz_off": int(R.L.pref_factor_nnz_off(f))})
        R.free_factor(f)
    R.free_graph(h)
    with open(OUT, "w") as fh:
        json.dump(out, fh, indent=1)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
