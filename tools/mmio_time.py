#!/usr/bin/env python3
"""Wall time of factor Matrix Market I/O: this library (all host threads) vs
the reference's write_factor / read_factor (oracle/_ref, single thread) on the
same factor; files compared byte for byte. One JSON line per size.
  python tools/mmio_time.py [--n 64 128]"""
import argparse, json, os, sys, tempfile, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle
import paper_2505_02977_b200 as P

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[64])
a = ap.parse_args()
R = oracle.Reference()
for n3 in a.n:
    g = P.gen_poisson3d(n3)
    h = R.graph_from_csr(g)
    f, _ = R.factor(h, P.ordering_random(g.n, 0).perm, 0, backend=R.LEFT, workers=os.cpu_count())
    arr = R.factor_arrays(f)
    fac = P.LdlFactor(arr["n"], arr["col_ptr"], arr["rows"], arr["values"], arr["diag"], arr["perm"])
    with tempfile.TemporaryDirectory() as d:
        o, r = os.path.join(d, "o"), os.path.join(d, "r")
        t = time.perf_counter(); P.write_factor(fac, o); tw = time.perf_counter() - t
        t = time.perf_counter(); R._chk(R.L.pref_write_factor(f, r.encode())); trw = time.perf_counter() - t
        same = all(open(o + e, "rb").read() == open(r + e, "rb").read() for e in (".G.mtx", ".D.mtx"))
        t = time.perf_counter(); back = P.read_factor(o); tr = time.perf_counter() - t
        fh = oracle.C.c_void_p()
        t = time.perf_counter(); R._chk(R.L.pref_read_factor(r.encode(), None, oracle.C.byref(fh))); trr = time.perf_counter() - t
        mb = (os.path.getsize(o + ".G.mtx") + os.path.getsize(o + ".D.mtx")) / 1e6
    print(json.dumps({"n3": n3, "lines": int(fac.nnz_off_diagonal() + fac.n), "mbytes": round(mb, 1),
                      "threads": os.cpu_count(), "write_s": tw, "ref_write_s": trw, "read_s": tr,
                      "ref_read_s": trr, "byte_identical": same,
                      "round_trip": bool(back.values.tobytes() == fac.values.tobytes())}), flush=True)
    R.free_factor(fh); R.free_factor(f); R.free_graph(h)
