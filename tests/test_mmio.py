"""Matrix Market text I/O against the UNMODIFIED reference
writers/readers (oracle/_ref, proj/src/matrix_market.cpp, proj/src/ordering.cpp):

  * files written by this library are byte-identical to the reference's
    (factor .G/.D, Laplacian, vectors incl. signed zeros / subnormals /
    extremes, permutations), at sizes that take the multi-threaded paths;
  * each side reads what the other wrote back to identical arrays;
  * malformed inputs fail with the reference's Errc and message.
Host-only (no GPU): runs in the CPU suite.
"""
import os

import numpy as np
import pytest

import oracle
import paper_2505_02977_b200 as P

pytestmark = pytest.mark.skipif(not oracle.Reference.available(), reason="oracle/_ref not built")


@pytest.fixture(scope="module")
def R():
    return oracle.Reference()


def ref_factor(R, g, seed=0):
    h = R.graph_from_csr(g)
    perm = P.ordering_random(g.n, seed).perm
    f, _ = R.factor(h, perm, seed, backend=R.SEQ)
    return h, f


def as_factor(a):
    return P.LdlFactor(a["n"], a["col_ptr"], a["rows"], a["values"], a["diag"], a["perm"])


def read(p):
    with open(p, "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("n3", [6, 40])  # 40^3: ~700k factor lines, parallel formatting and parsing
def test_factor_files_byte_identical_and_round_trip(R, tmp_path, n3):
    g = P.gen_poisson3d(n3, "contrast", 1e-3, 1e4, 3)
    h, f = ref_factor(R, g, 5)
    a = R.factor_arrays(f)
    ours, theirs = str(tmp_path / "ours"), str(tmp_path / "ref")
    P.write_factor(as_factor(a), ours)
    R._chk(R.L.pref_write_factor(f, theirs.encode()))
    for ext in (".G.mtx", ".D.mtx"):
        assert read(ours + ext) == read(theirs + ext), ext
    # permutation file, then both readers on the reference's files
    P.write_permutation(ours + ".perm.txt", P.Ordering(a["perm"]))
    R._chk(R.L.pref_write_permutation((theirs + ".perm.txt").encode(), g.n, a["perm"].ctypes.data))
    assert read(ours + ".perm.txt") == read(theirs + ".perm.txt")
    back = P.read_factor(theirs, theirs + ".perm.txt")
    assert back.same_values(as_factor(a))
    fh = oracle.C.c_void_p()
    R._chk(R.L.pref_read_factor(ours.encode(), (ours + ".perm.txt").encode(), oracle.C.byref(fh)))
    assert as_factor(R.factor_arrays(fh)).same_values(as_factor(a))
    assert P.read_factor(ours).perm.tolist() == list(range(g.n))  # no perm file: identity
    R.free_factor(fh)
    R.free_factor(f)
    R.free_graph(h)


@pytest.mark.parametrize("name,build", [
    ("poisson3d_contrast", lambda: P.gen_poisson3d(7, "contrast", 1e-3, 1e4, 1)),
    ("poisson27", lambda: P.gen_poisson27(6, 1)),
    ("random_connected", lambda: P.gen_random_connected(3000, 9000, 4, False)),
    ("rmat_12", lambda: P.gen_rmat(12, 16, 0)),
])
def test_laplacian_write_identical_and_read_back(R, tmp_path, name, build):
    g = build()
    h = R.graph_from_csr(g)
    ours, theirs = str(tmp_path / "ours.mtx"), str(tmp_path / "ref.mtx")
    P.write_matrix_market(ours, g)
    R._chk(R.L.pref_write_matrix_market(theirs.encode(), h))
    assert read(ours) == read(theirs)
    back = P.read_laplacian(theirs)
    assert np.array_equal(back.ptr, g.ptr) and np.array_equal(back.adj, g.adj)
    assert back.w.tobytes() == g.w.tobytes() and back.wdeg.tobytes() == g.wdeg.tobytes()
    hh = oracle.C.c_void_p()
    R._chk(R.L.pref_read_laplacian(ours.encode(), oracle.C.byref(hh)))
    _, ptr, _, w, _ = R.csr(hh)
    assert np.array_equal(ptr, g.ptr) and w.tobytes() == g.w.tobytes()
    R.free_graph(hh)
    R.free_graph(h)


def test_vector_special_values(R, tmp_path):
    rng = np.random.default_rng(0)
    v = np.concatenate([[0.0, -0.0, 5e-324, -2.2250738585072014e-308, 1.7976931348623157e308, 0.1, 1 / 3,
                         1e-5, 123456789.0, 1e16, 1e17, -1e-100],
                        rng.standard_normal(200000) * 10.0 ** rng.integers(-300, 300, 200000)])
    ours, theirs = str(tmp_path / "o.mtx"), str(tmp_path / "r.mtx")
    P.write_vector(ours, v)
    R._chk(R.L.pref_write_vector(theirs.encode(), len(v), v.ctypes.data))
    assert read(ours) == read(theirs)
    assert P.read_vector(theirs).tobytes() == v.tobytes()
    out = np.empty(len(v)); n = oracle.C.c_int64()
    R._chk(R.L.pref_read_vector(ours.encode(), len(v), out.ctypes.data, oracle.C.byref(n)))
    assert n.value == len(v) and out.tobytes() == v.tobytes()


BAD = {
    "missing": None,
    "empty.mtx": "",
    "nobanner.mtx": "hello\n1 1 1\n1 1 1.0\n",
    "array.mtx": "%%MatrixMarket matrix array real general\n2 1\n1\n2\n",
    "badsize.mtx": "%%MatrixMarket matrix coordinate real symmetric\n% c\n\n2 x 3\n",
    "truncated.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 1.0\n2 1 -1.0\n",
    "oob.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n3 1 -1.0\n",
    "malformed.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 1.0\n2 1 abc\n",
    "inf.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 2\n1 1 inf\n2 1 -1\n",
    "asym.mtx": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1\n2 2 1\n2 1 -1\n",
    "positive.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 -1\n2 2 -1\n2 1 1\n",
    "rowsum.mtx": "%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2\n2 2 1\n2 1 -1\n",
    "notsquare.mtx": "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 1 1\n",
    "ok_dups.mtx": "%%MatrixMarket matrix coordinate real general\n3 3 8\n1 1 2\n2 2 1.5\n3 3 0.5\n"
                   "2 1 -0.5\n2 1 -0.5\n1 2 -1\n3 1 -1\n1 3 -0.5\n+3 +1 +0.5\n",
}


def code_and_message(fn):
    try:
        fn()
        return 0, ""
    except P.Error as e:
        return int(e.code), str(e)


@pytest.mark.parametrize("name", sorted(BAD))
def test_laplacian_reader_errors_match_reference(R, tmp_path, name):
    path = str(tmp_path / name)
    if BAD[name] is not None:
        with open(path, "w") as fh:
            fh.write(BAD[name])
    code, msg = code_and_message(lambda: P.read_laplacian(path))
    hh = oracle.C.c_void_p()
    rc = R.L.pref_read_laplacian(path.encode(), oracle.C.byref(hh))
    assert code == rc, (name, msg, R.L.pref_last_error())
    if rc:
        assert R.L.pref_last_error().decode() in msg, (msg, R.L.pref_last_error())
    else:
        _, ptr, _, w, _ = R.csr(hh)
        g = P.read_laplacian(path)
        assert np.array_equal(ptr, g.ptr) and w.tobytes() == g.w.tobytes()
        R.free_graph(hh)


FACTOR_BAD = {
    "hdr": ("%%MatrixMarket matrix coordinate real symmetric\n2 2 1\n2 1 0.5\n", "%%MatrixMarket matrix array real general\n2 1\n1\n1\n"),
    "upper": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 0.5\n", "%%MatrixMarket matrix array real general\n2 1\n1\n1\n"),
    "short": ("%%MatrixMarket matrix coordinate real general\n2 2 2\n2 1 0.5\n", "%%MatrixMarket matrix array real general\n2 1\n1\n1\n"),
    "diaglen": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 0.5\n", "%%MatrixMarket matrix array real general\n3 1\n1\n1\n1\n"),
    "diagbad": ("%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 0.5\n", "%%MatrixMarket matrix array real general\n2 1\n1\nx\n"),
    "ok": ("%%MatrixMarket matrix coordinate real general\n% c\n3 3 3\n3 1 0.25\n2 1 -0.5\n3 2 1e-3\n",
           "%%MatrixMarket matrix array real general\n3 1\n1\n% c\n2\n0\n"),
}


@pytest.mark.parametrize("name", sorted(FACTOR_BAD))
def test_factor_reader_errors_match_reference(R, tmp_path, name):
    stem = str(tmp_path / name)
    gtxt, dtxt = FACTOR_BAD[name]
    with open(stem + ".G.mtx", "w") as fh:
        fh.write(gtxt)
    with open(stem + ".D.mtx", "w") as fh:
        fh.write(dtxt)
    code, msg = code_and_message(lambda: P.read_factor(stem))
    fh = oracle.C.c_void_p()
    rc = R.L.pref_read_factor(stem.encode(), None, oracle.C.byref(fh))
    assert code == rc, (name, msg, R.L.pref_last_error())
    if rc:
        assert R.L.pref_last_error().decode() in msg
    else:
        assert as_factor(R.factor_arrays(fh)).same_values(P.read_factor(stem))
        R.free_factor(fh)


def test_permutation_errors(tmp_path):
    p = str(tmp_path / "perm.txt")
    with open(p, "w") as fh:
        fh.write("0\n1\n1\n")
    assert code_and_message(lambda: P.ordering_from_file(p, 3))[0] == P.Errc.not_a_permutation
    assert code_and_message(lambda: P.ordering_from_file(p, 4))[0] == P.Errc.not_a_permutation
    assert code_and_message(lambda: P.ordering_from_file(str(tmp_path / "none"), 3))[0] == P.Errc.io_error
