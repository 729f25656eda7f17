"""GPU: the C++ drop-in (csrc/shim/parac_gpu_shim.hpp) called from a program
built against the reference's own headers and library (oracle/shim_check.cpp):
parac::factor_gpu same_values factor_randomized, FactorStats equal,
pcg_solve_gpu within 10% of pcg_solve, bit-identical apply_preconditioner /
laplacian_apply, and the reference's Errc codes thrown as parac::Error."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "shim_check")

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("side", [12, 32])
def test_cpp_shim_against_reference(side):
    if not os.path.exists(BIN):
        pytest.fail("oracle/_ref/shim_check not built (make -C oracle shim, in the build container)")
    out = subprocess.run([BIN, str(side)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ALL PASS" in out.stdout
