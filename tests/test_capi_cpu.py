"""CPU tests of the C-ABI library: it loads without a GPU, exports every
symbol include/hexmg_b200.h declares, and its host-side setup (basis,
geometry, constraints, traction load) matches the golden fixtures / oracle.
No device computation here."""
import os
import re

import numpy as np
import pytest

from oracle import hexmg_np as H

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hexmg_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(hxg_\w+)\(", src, re.M)))


@pytest.fixture(scope="module")
def L():
    from paper_2204_01722_b200 import capi
    if not os.path.exists(capi.library_path):
        pytest.fail("libhexmg_b200.so not built (run __graft_entry__.build())")
    return capi.lib()


def test_exports_every_declared_symbol(L):
    from paper_2204_01722_b200 import capi
    syms = declared_symbols()
    assert len(syms) > 40
    for s in syms:
        assert hasattr(L, s), s
        assert s in capi.SIGNATURES, f"{s} missing from the ctypes binding"


def test_version(L):
    assert b"sm_100a" in L.hxg_version()


@pytest.mark.parametrize("p,q", [(1, 2), (2, 3), (3, 4), (4, 5), (1, 3), (1, 4), (1, 5), (2, 4), (2, 5)])
def test_host_basis_matches_golden(L, p, q):
    from paper_2204_01722_b200.hexmg import build_lagrange_basis
    g = np.load(os.path.join(GOLD, "basis.npz"))
    b = build_lagrange_basis(p, q)
    for k in ("nodes", "points", "weights", "interp", "deriv", "pinv", "colloc"):
        np.testing.assert_allclose(getattr(b, k), g[f"p{p}q{q}_{k}"], atol=2e-15, rtol=0)


@pytest.mark.parametrize("order,cells,ext", [(2, (4, 2, 2), (2.0, 1.0, 1.0)), (3, (2, 2, 2), (1.0, 1.0, 1.0)),
                                             (1, (3, 2, 2), (1.7, 0.9, 1.3))])
def test_host_geometry_constraints_load(L, order, cells, ext):
    from paper_2204_01722_b200 import hexmg as G
    P = H.make_problem(ext, cells, order, traction_face=1, traction=(0, 0, -0.02))
    dx, w = G.geometric_factors(ext, cells, order, order + 1)
    np.testing.assert_allclose(dx, P.op.dxidX, atol=1e-13, rtol=0)
    np.testing.assert_allclose(w, P.op.weight, atol=1e-15, rtol=1e-13)
    m, fm = G.constraint_mask(cells, order, ("-x",))
    assert fm == 1
    assert np.array_equal(m, P.op.mask)
    load = G.traction_load(ext, cells, order, order + 1, "+x", (0, 0, -0.02))
    np.testing.assert_allclose(load, P.load, atol=1e-16, rtol=1e-13)


def test_invalid_arguments_raise(L):
    from paper_2204_01722_b200 import hexmg as G
    from paper_2204_01722_b200.capi import HxgError
    with pytest.raises(HxgError):
        G.build_lagrange_basis(2, 2)  # q < p + 1 (basis.hpp:137-138)
    with pytest.raises(HxgError):
        G.build_lagrange_basis(0, 2)
    with pytest.raises(ValueError):
        G.lame_from_young_poisson(1.0, 0.5)


def test_dropin_binary_links():
    """The C++ drop-in test binary (oracle/Makefile target, built from the
    reference headers + include/hexmg_b200.hpp) resolves libhexmg_b200.so
    in-tree; it runs under -m gpu (tests/test_gpu_dropin.py)."""
    import subprocess
    exe = os.path.join(ROOT, "oracle", "_ref", "test_dropin")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/test_dropin not built (needs /root/reference)")
    out = subprocess.run(["ldd", exe], capture_output=True, text=True).stdout
    assert "libhexmg_b200.so" in out and "not found" not in out, out
