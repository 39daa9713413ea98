"""Inexact coarse mode (hxg_mg_set_coarse_mode 4, csrc/hcoarse.cu): the p = 1
level solved by one Galerkin h-multigrid V-cycle instead of the reference's
exact SimplicialLLT (coarse_solver.hpp:16-47).  A documented deviation, so
there is no reference output to match; the tests pin what it must satisfy:

* every h-level matrix is the Galerkin product P~^T A P~ of the level above
  (trilinear P, constrained fine rows / coarse columns dropped, identity on
  the constrained coarse rows), checked against scipy from the exported CSRs;
* the p-MG V-cycle stays a symmetric operator (PCG-valid);
* PCG reaches the same rtol as the exact mode with at most two more
  iterations, and the same solution;
* the fused residual path feeds it (Newton converges like the exact mode)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
sp = pytest.importorskip("scipy.sparse")

pytestmark = pytest.mark.gpu


def _cube(order, n, **kw):
    from paper_2204_01722_b200.hexmg import FemProblem
    return FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",),
                      traction_face="+x", traction=(0, 0, -0.02), **kw)


def _prolongation(npd_f, npd_c, mask_f):
    """Trilinear P (3 n_f x 3 n_c) with the constrained fine rows removed."""
    rows, cols, vals = [], [], []
    nf = npd_f[0] * npd_f[1] * npd_f[2]
    for node in range(nf):
        g = (node % npd_f[0], (node // npd_f[0]) % npd_f[1], node // (npd_f[0] * npd_f[1]))
        opts = []
        for d in range(3):
            opts.append([(g[d] // 2, 1.0)] if g[d] % 2 == 0 else [((g[d] - 1) // 2, 0.5), ((g[d] + 1) // 2, 0.5)])
        for cz, wz in opts[2]:
            for cy, wy in opts[1]:
                for cx, wx in opts[0]:
                    cn = cx + npd_c[0] * (cy + npd_c[1] * cz)
                    for c in range(3):
                        if mask_f[3 * node + c]:
                            continue
                        rows.append(3 * node + c)
                        cols.append(3 * cn + c)
                        vals.append(wx * wy * wz)
    nc = npd_c[0] * npd_c[1] * npd_c[2]
    return sp.csr_matrix((vals, (rows, cols)), shape=(3 * nf, 3 * nc))


@pytest.mark.parametrize("order,n", [(2, 16), (2, 13)])
def test_hmg_levels_are_galerkin_products(order, n):
    prob = _cube(order, n)
    prob.op.apply_residual(torch.zeros(prob.size(), dtype=torch.float64, device="cuda"))
    mg = prob.hierarchy
    mg.set_coarse_mode("hmg")
    mg.setup_numeric()
    L = mg.hmg_levels()
    assert L >= 2
    cells = [n, n, n]
    for lev in range(L - 1):
        rp, cols, vals, mask = mg.hmg_level_csr(lev)
        A = sp.csr_matrix((vals, cols, rp), shape=(len(rp) - 1,) * 2)
        rp1, cols1, vals1, mask1 = mg.hmg_level_csr(lev + 1)
        A1 = sp.csr_matrix((vals1, cols1, rp1), shape=(len(rp1) - 1,) * 2).toarray()
        ccells = [(c + 1) // 2 for c in cells]
        npd_f, npd_c = [c + 1 for c in cells], [c + 1 for c in ccells]
        P = _prolongation(npd_f, npd_c, mask)
        free = sp.diags((mask == 0).astype(float))
        G = (P.T @ (free @ A @ free) @ P).toarray()
        # coarse DoFs with an empty P~ column are constrained: identity rows
        empty = np.asarray(abs(P).sum(axis=0)).ravel() == 0
        assert np.array_equal(empty, mask1 != 0)
        G[empty, :] = 0.0
        G[:, empty] = 0.0
        G[empty, empty] = 1.0
        assert np.abs(A1 - G).max() <= 1e-12 * np.abs(G).max()
        cells = ccells


def test_hmg_vcycle_is_symmetric():
    prob = _cube(2, 16)
    N = prob.size()
    prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
    mg = prob.hierarchy
    mg.set_coarse_mode("hmg")
    mg.setup_numeric()
    g = torch.Generator(device="cpu").manual_seed(7)
    m = torch.from_numpy(prob.mask == 0).cuda()
    u = (torch.rand(N, generator=g, dtype=torch.float64) - 0.5).cuda() * m
    v = (torch.rand(N, generator=g, dtype=torch.float64) - 0.5).cuda() * m
    a = torch.dot(u, mg.v_cycle(v)).item()
    b = torch.dot(v, mg.v_cycle(u)).item()
    assert abs(a - b) <= 1e-12 * max(abs(a), abs(b))
    # deterministic: bitwise equal run to run
    assert torch.equal(mg.v_cycle(v), mg.v_cycle(v))


@pytest.mark.parametrize("order,n", [(2, 16), (2, 24), (3, 12), (4, 10)])
def test_hmg_pcg_reaches_the_exact_solution(order, n):
    from paper_2204_01722_b200.hexmg import cg_solve
    prob = _cube(order, n)
    N = prob.size()
    f = prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
    mg = prob.hierarchy
    mg.set_coarse_mode("auto")
    mg.setup_numeric()
    ex = cg_solve(prob.op, -f, rtol=1e-8, precond="mg", mg=mg)
    mg.set_coarse_mode("hmg")
    mg.setup_numeric()
    assert mg.hmg_levels() >= 1
    ih = cg_solve(prob.op, -f, rtol=1e-8, precond="mg", mg=mg)
    assert ih["converged"] and ex["converged"]
    assert ih["iterations"] <= ex["iterations"] + 2
    rel = (torch.linalg.norm(ih["x"] - ex["x"]) / torch.linalg.norm(ex["x"])).item()
    assert rel < 1e-7


def test_hmg_newton_matches_exact_mode():
    from paper_2204_01722_b200.hexmg import FemProblem
    kw = dict(extents=(2, 1, 1), cells=(16, 8, 8), order=2, fixed_faces=("-x",),
              traction_face="+x", traction=(-0.05, 0, 0))
    ex = FemProblem(**kw).solve(load_steps=2)
    prob = FemProblem(**kw)
    prob.hierarchy.set_coarse_mode("hmg")
    ih = prob.solve(load_steps=2)
    assert ih["converged"] and ih["newton_iterations"] == ex["newton_iterations"]
    rel = (torch.linalg.norm(ih["u"] - ex["u"]) / torch.linalg.norm(ex["u"])).item()
    assert rel < 1e-8
