"""The C++ drop-in (include/hexmg_b200.hpp) used the way a reference-side
caller would: tests/cpp/test_dropin.cpp builds the problem with the
UNMODIFIED reference headers (BoxMesh, Basis1D, GeometricFactors,
Constraints, traction load; problem.hpp:19-58), constructs
hexmg::b200::MatrixFreeOperator with the reference constructor signature
(operator.hpp:72-97) and compares it with hexmg::MatrixFreeOperator
(residual 1e-11, Jacobian / diagonal / energy 1e-12), then
hexmg::b200::build_hierarchy + cg_solve against the reference's
(multigrid.hpp:212, cg.hpp:81; iterations within +-1, solution 1e-7), and
the reference exception types (StateNotInitializedError, InvertedElementError
at the reference's element / point).  The binary is built by oracle/Makefile
in the container that has /root/reference and travels to the GPU box."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "test_dropin")

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/test_dropin not built")]


@pytest.mark.parametrize("order,n", [(2, 8), (3, 6), (4, 4), (2, 16)])
def test_dropin_matches_reference(order, n):
    p = subprocess.run([BIN, str(order), str(n), str(os.cpu_count() or 1)], capture_output=True,
                       text=True, timeout=600)
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert lines, p.stdout + p.stderr
    r = json.loads(lines[-1])
    assert r["ok"], r
    assert p.returncode == 0, r
