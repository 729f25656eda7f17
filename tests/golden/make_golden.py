"""Generate tests/golden/golden.json from the UNMODIFIED reference build
(oracle/_ref/libparac_ref.so, compiled from /root/reference/proj/src by
oracle/Makefile). Run in the dev container:  python tests/golden/make_golden.py

Every value here is produced by the reference's own public API; the tests then
pin both the C restatement (oracle/rchol_oracle.c) and the CUDA path to it
without needing /root/reference at run time.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.json")


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()[:32]


def main() -> None:
    oracle.build(reference=True)
    R = oracle.Reference()
    gold = {"_source": "oracle/_ref (unmodified reference, proj/src/*.cpp)", "factors": [],
            "graphs": [], "orderings": [], "pcg": [], "precond": []}

    def add_factor(name, h, perm, seed, backend=0, workers=1, levels=True):
        f, _ = R.factor(h, perm, seed, backend=backend, workers=workers, stats=True)
        arr = R.factor_arrays(f)
        st = R.factor_stats(f)
        entry = {
            "name": name, "seed": seed, "n": arr["n"],
            "checksum": f"{R.checksum(f):016x}",
            "nnz_off": int(len(arr["rows"])),
            "total_fills": int(st["total_fills"]),
            "stats_digest": digest(st["merged_degree"], st["samples_emitted"], st["fills_received"]),
            "perm_digest": digest(perm),
            "depth": int(R.L.pref_schedule_depth(f)),
        }
        if arr["n"] <= 64:
            entry["arrays"] = {k: arr[k].tolist() for k in ("col_ptr", "rows", "values", "diag")}
        gold["factors"].append(entry)
        R.free_factor(f)

    # Reference known-answer cases (proj/tests/test_factor_seq.cpp:14-54)
    def edges_graph(n, edges):
        a = np.array([e[0] for e in edges], np.int32)
        b = np.array([e[1] for e in edges], np.int32)
        w = np.array([e[2] for e in edges], np.float64)
        h = oracle.vp()
        R._chk(R.L.pref_graph_from_edges(n, len(edges), a.ctypes.data, b.ctypes.data,
                                         w.ctypes.data, oracle.C.byref(h)))
        return h

    p3 = edges_graph(3, [(0, 1, 1.0), (1, 2, 1.0)])
    k3 = edges_graph(3, [(0, 1, 1.0), (0, 2, 1.0), (1, 2, 1.0)])
    ident3 = np.arange(3, dtype=np.int32)
    add_factor("p3", p3, ident3, 0)
    for s in (0, 7, 123456):
        add_factor(f"k3_s{s}", k3, ident3, s)
    for leaves in (3, 8):
        star = edges_graph(leaves + 1, [(0, v, 1.0) for v in range(1, leaves + 1)])
        add_factor(f"star{leaves}", star, np.arange(leaves + 1, dtype=np.int32), 0)
    for n in (2, 5, 9):
        ring = edges_graph(n, [(v, v + 1, 1.0) for v in range(n - 1)] + ([(0, n - 1, 1.0)] if n > 2 else []))
        for s in range(4):
            add_factor(f"ring{n}_s{s}", ring, R.ordering_random(n, s), s)

    # Random graph corpus (proj/tests/test_factor_par.cpp:20-65, acceptance.cpp:154-210)
    for seed in range(3):
        h = R.random_connected(200, 400, seed * 31 + 1)
        add_factor(f"rc200_s{seed}_random", h, R.ordering_random(200, seed), seed)
        add_factor(f"rc200_s{seed}_nnz", h, R.ordering_nnz_sort(h, seed), seed + 1)
    for seed in range(6):
        h = R.random_connected(50, 80, seed)
        add_factor(f"rc50_s{seed}", h, R.ordering_random(50, seed), seed)
    multi = R.random_components(120, 4, 60, 5)
    add_factor("components120", multi, R.ordering_random(120, 9), 2)
    for seed in range(4):
        h = R.random_components(3000, 3, 9000, seed)
        add_factor(f"components3000_s{seed}", h, R.ordering_random(3000, seed), seed)

    # Poisson grids (BASELINE.md §3 checksums at 32^3 / 64^3)
    for n in (8, 16, 32, 64):
        h = R.poisson3d(n)
        N = n ** 3
        add_factor(f"poisson{n}_random0", h, R.ordering_random(N, 0), 0)
        if n in (16, 32):
            add_factor(f"poisson{n}_nnz0", h, R.ordering_nnz_sort(h, 0), 0)
            add_factor(f"poisson{n}_random1", h, R.ordering_random(N, 1), 1)
    hc = R.poisson3d(12, variant=2, contrast=1e4, seed=3)
    add_factor("poisson12_contrast", hc, R.ordering_random(12 ** 3, 0), 0)
    ha = R.poisson3d(12, variant=1, eps=1e-3)
    add_factor("poisson12_aniso", ha, R.ordering_nnz_sort(ha, 0), 0)

    # Generator + ordering digests (host builders must equal the reference's)
    for name, h in (("poisson16", R.poisson3d(16)), ("poisson12_contrast", hc),
                    ("poisson12_aniso", ha), ("rc200_1", R.random_connected(200, 400, 1)),
                    ("components120", multi)):
        n, ptr, adj, w, wdeg = R.csr(h)
        gold["graphs"].append({"name": name, "n": int(n), "digest": digest(ptr, adj, w, wdeg)})
    for n, seed in ((1000, 0), (4096, 5), (32768, 0)):
        gold["orderings"].append({"kind": "random", "n": n, "seed": seed,
                                  "digest": digest(R.ordering_random(n, seed))})
    gold["orderings"].append({"kind": "nnz_sort", "graph": "rc200_1", "seed": 3,
                              "digest": digest(R.ordering_nnz_sort(R.random_connected(200, 400, 1), 3))})

    # PCG (proj/tests/test_solver.cpp:115-126, acceptance.cpp:215-251)
    def add_pcg(name, h, perm, seed, rhs_seed, tol):
        f, _ = R.factor(h, perm, seed)
        n = R.L.pref_graph_n(h)
        b = np.empty(n, np.float64)
        R._chk(R.L.pref_make_rhs(h, 1, rhs_seed, b.ctypes.data))
        x = np.empty(n, np.float64)
        it, conv = oracle.C.c_int(), oracle.C.c_int()
        rel, rec, sec = oracle.f64(), oracle.f64(), oracle.f64()
        R._chk(R.L.pref_pcg(h, f, b.ctypes.data, tol, 1000, x.ctypes.data, oracle.C.byref(it),
                            oracle.C.byref(rel), oracle.C.byref(rec), oracle.C.byref(conv),
                            oracle.C.byref(sec)))
        gold["pcg"].append({"name": name, "seed": seed, "rhs_seed": rhs_seed, "tol": tol,
                            "iterations": it.value, "relative_residual": rel.value,
                            "recurrence_residual": rec.value, "converged": bool(conv.value),
                            "rhs_digest": digest(b), "x_digest": digest(x)})
        R.free_factor(f)

    h12 = R.poisson3d(12)
    add_pcg("poisson12_nnz", h12, R.ordering_nnz_sort(h12, 0), 0, 1, 1e-6)
    h32 = R.poisson3d(32)
    add_pcg("poisson32_nnz", h32, R.ordering_nnz_sort(h32, 0), 0, 0, 1e-6)
    add_pcg("poisson32_random_1e-8", h32, R.ordering_random(32 ** 3, 0), 0, 0, 1e-8)
    h16 = R.poisson3d(16)
    add_pcg("poisson16_random_1e-8", h16, R.ordering_random(16 ** 3, 0), 0, 0, 1e-8)

    # apply_preconditioner digest on a random factor (bit-exact target)
    h = R.random_connected(300, 700, 4)
    perm = R.ordering_random(300, 2)
    f, _ = R.factor(h, perm, 3)
    r = np.empty(300, np.float64)
    R._chk(R.L.pref_make_rhs(h, 1, 9, r.ctypes.data))
    z = np.empty(300, np.float64)
    R._chk(R.L.pref_apply_preconditioner(f, r.ctypes.data, z.ctypes.data))
    gold["precond"].append({"name": "rc300_s4", "seed": 3, "rhs_seed": 9, "z_digest": digest(z)})
    R.free_factor(f)

    with open(OUT, "w") as fh:
        json.dump(gold, fh, indent=1)
    print(f"wrote {OUT}: {len(gold['factors'])} factors, {len(gold['pcg'])} pcg")


if __name__ == "__main__":
    main()
