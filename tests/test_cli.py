"""Host-side behaviour of the parac-compatible runner (paper_2505_02977_b200/cli.py)
that needs no GPU: generator-spec parsing (src/generators.cpp:67-108), the gen
command's Matrix Market output (byte-identical to the reference writer, via
the oracle), exit codes 10 + Errc (parac_cli.cpp:39), and the CSV / number
formatting of parac-bench-v1 rows (parac_cli.cpp:182-193, :425-441)."""
import numpy as np
import pytest

import oracle
import paper_2505_02977_b200 as P
from paper_2505_02977_b200 import cli


def test_parse_gen_spec_matches_generators():
    g = cli.parse_gen_spec("poisson3d:n=5,variant=contrast,epsilon=2e-3,contrast=100,seed=7")
    want = P.gen_poisson3d(5, "contrast", 2e-3, 100.0, 7)
    assert np.array_equal(g.ptr, want.ptr) and g.w.tobytes() == want.w.tobytes()
    assert cli.parse_gen_spec("poisson2d:n=6").n == 36
    assert cli.parse_gen_spec("poisson27:n=4,seed=1").n == 64
    assert cli.parse_gen_spec("rmat:scale=8,edge_factor=4,seed=0").n == 256


@pytest.mark.parametrize("spec", ["cube:n=4", "poisson3d:n", "poisson3d:n=x", "poisson3d:n=4,variant=odd",
                                  "poisson3d:n=4,bogus=1", "poisson3d:n=4,epsilon=0"])
def test_parse_gen_spec_errors(spec):
    with pytest.raises(cli.CliError) as e:
        cli.parse_gen_spec(spec)
    assert e.value.code == int(P.Errc.parse_error)


def test_exit_codes_without_gpu(tmp_path):
    assert cli.main(["factor", "--gen", "poisson3d:n=4", "--backend", "seq"]) == 15
    assert cli.main(["factor", "--input", "a.mtx", "--gen", "poisson3d:n=4", "--backend", "par-left"]) == 15
    assert cli.main(["gen", "--gen", "poisson3d:n=4,foo=1", "--output", str(tmp_path / "x.mtx")]) == 15


@pytest.mark.skipif(not oracle.Reference.available(), reason="oracle/_ref not built")
def test_gen_command_writes_reference_bytes(tmp_path, capsys):
    out = str(tmp_path / "g.mtx")
    assert cli.main(["gen", "--gen", "poisson3d:n=6,variant=anisotropic,epsilon=0.01", "--output", out]) == 0
    assert "216 vertices" in capsys.readouterr().out
    R = oracle.Reference()
    h = R.poisson3d(6, 1, 0.01, 1e4, 0)
    ref = str(tmp_path / "r.mtx")
    R._chk(R.L.pref_write_matrix_market(ref.encode(), h))
    assert open(out, "rb").read() == open(ref, "rb").read()
    g = P.read_laplacian(out)
    assert g.n == 216
    R.free_graph(h)


def test_number_and_field_formatting():
    # std::ostream << double (default precision 6) == printf %g
    assert cli._g(0.0123456789) == "0.0123457"
    assert cli._g(1.5e-9) == "1.5e-09"
    assert cli._g(3.0) == "3"
    assert cli._csv_field("poisson3d:n=4") == "poisson3d:n=4"
    assert cli._csv_field('a,b"c') == '"a,b""c"'


def test_fill_ratio_definition():
    # etree.cpp:137-142: 2 nnz(G) / (nnz_off(L) + n); P3 gives 10/7 (tests/test_cli.cpp:45-58)
    g = P.LaplacianGraph.from_edges(3, [(0, 1, 1.0), (1, 2, 1.0)])
    f = P.LdlFactor(3, np.array([0, 1, 2, 2]), np.array([1, 2], np.int32), np.array([-1.0, -1.0]),
                    np.array([1.0, 1.0, 0.0]), np.arange(3, dtype=np.int32))
    assert cli.fill_ratio(g, f) == pytest.approx(10 / 7)
