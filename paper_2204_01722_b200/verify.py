"""Invariant suite (run_verification, verify.hpp:63-285) on this framework:
the same fourteen named checks, instances, seeds and thresholds, evaluated
through the device operator, hierarchy and assembled representation.  The
jacobian_perturbation hook (verify.hpp:20-25) must make jacobian-fd fail.

Each result is (name, passed, detail); the detail strings follow the
reference's wording."""
from __future__ import annotations

import numpy as np
import torch

from .hexmg import (STATE_SCALARS, AssembledOperator, FemProblem, build_lagrange_basis,
                    geometric_factors)


def random_field(n, seed, scale):
    """verify_detail::random_field (verify.hpp:29-34): mt19937(seed) raw
    32-bit draws mapped to scale * (2 u - 1)."""
    raw = np.random.RandomState(seed).randint(0, 2**32, size=n, dtype=np.uint64).astype(np.float64)
    return scale * (2.0 * (raw * (1.0 / 4294967296.0)) - 1.0)


def rel_diff(a, b):
    num = float(np.sum((a - b) ** 2))
    den = float(np.sum(b * b))
    return float(np.sqrt(num / den)) if den > 0 else float(np.sqrt(num))


def _fd(v):
    return "%.17g" % v


def _coo_to_csr(rows, cols, vals, n):
    """build_coo_template + fill_from_coo semantics (assembly.hpp:70-130):
    negative indices discarded, duplicates summed."""
    keep = [(r, c, v) for r, c, v in zip(rows, cols, vals) if r >= 0 and c >= 0]
    acc = {}
    for r, c, v in keep:
        acc[(r, c)] = acc.get((r, c), 0.0) + v
    return acc


def run_verification(jacobian_perturbation=0.0):
    res = []

    def check(name, ok, detail):
        res.append((name, bool(ok), detail))

    # Quadrature exactness up to degree 2q - 1 (q = 1 is the midpoint rule).
    worst = 0.0
    for q in range(1, 6):
        if q == 1:
            pts, wts = np.array([0.0]), np.array([2.0])
        else:
            b = build_lagrange_basis(1, q)
            pts, wts = b.points, b.weights
        for k in range(2 * q):
            exact = 2.0 / (k + 1) if k % 2 == 0 else 0.0
            worst = max(worst, abs(float(np.sum(wts * pts**k)) - exact))
    check("quadrature-exactness", worst < 1e-13, "max error " + _fd(worst))

    # Basis row sums: interpolation rows to 1, derivative rows to 0.
    worst = 0.0
    for p in range(1, 5):
        b = build_lagrange_basis(p)
        worst = max(worst, float(np.max(np.abs(b.interp.sum(1) - 1.0))),
                    float(np.max(np.abs(b.deriv.sum(1)))))
    check("basis-row-sums", worst < 1e-13, "max deviation " + _fd(worst))

    # Sum-factorized gradient adjoint identity on random data (p = 3).
    b = build_lagrange_basis(3)
    N, Q, ne = 4, b.q, 2
    x = random_field(ne * 3 * N**3, 11, 1.0).reshape(ne, 3, N, N, N)  # (e, c, k, j, i)
    B, D = b.interp, b.deriv
    gx = np.stack([np.einsum("xi,yj,zk,eckji->eczyx", *t, x)
                   for t in ((D, B, B), (B, D, B), (B, B, D))], 2)  # (e, c, d, z, y, x)
    y = random_field(gx.size, 12, 1.0).reshape(gx.shape)
    yt = sum(np.einsum("xi,yj,zk,eczyx->eckji", *t, y[:, :, d])
             for d, t in enumerate(((D, B, B), (B, D, B), (B, B, D))))
    lhs, rhs = float(np.sum(gx * y)), float(np.sum(x * yt))
    err = abs(lhs - rhs) / max(1.0, abs(lhs))
    check("basis-grad-adjoint", err < 1e-13, "inner product gap " + _fd(err))

    # Gather/scatter roundtrip equals the multiplicity scaling (device).
    pr = FemProblem(extents=(1.0, 1.0, 1.0), cells=(2, 2, 2), order=2, fixed_faces=())
    n = pr.size()
    u = torch.from_numpy(random_field(n, 21, 1.0)).cuda()
    ev = pr.op.gather(u, pr.num_elements, 27)
    out = torch.zeros_like(u)
    pr.op.scatter_add(ev, out)
    ones = torch.ones_like(u)
    mult = torch.zeros_like(u)
    pr.op.scatter_add(pr.op.gather(ones, pr.num_elements, 27), mult)
    worst = float((out - mult * u).abs().max())
    check("restriction-roundtrip", worst < 1e-12, "max deviation " + _fd(worst))

    # Geometric factor inverse consistency: dX/dxi (affine box: diag(h / 2))
    # times the library's dxi/dX.
    ext, cells = (1.7, 0.9, 1.3), (2, 1, 2)
    dx, _ = geometric_factors(ext, cells, 2, 3)
    dXdxi = np.diag([ext[d] / (2.0 * cells[d]) for d in range(3)])
    prod = np.einsum("ij,...jk->...ik", dXdxi, np.asarray(dx).reshape(-1, 3, 3))
    worst = float(np.max(np.abs(prod - np.eye(3))))
    check("geometry-inverse", worst < 1e-12, "max deviation " + _fd(worst))

    # Shared setup for the operator-level checks: bar_config(2, 1).
    prob = FemProblem(extents=(2.0, 1.0, 1.0), cells=(2, 1, 1), order=2, fixed_faces=("-x",),
                      traction_face="+x", traction=(0.0, 0.0, -0.02))
    op = prob.op
    op.set_jacobian_perturbation(jacobian_perturbation)
    n = prob.size()
    mask = np.asarray(prob.mask) != 0
    u = np.where(mask, 0.0, random_field(n, 31, 0.02))
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    host = lambda t: t.detach().cpu().numpy()  # noqa: E731
    f = host(op.apply_residual(cu(u)))

    du = np.where(mask, 0.0, random_field(n, 32, 1.0))
    ju = host(op.apply_jacobian(cu(du)))
    h = 1e-6
    fp = host(op.apply_residual(cu(u + h * du)))
    fm = host(op.apply_residual(cu(u - h * du)))
    err = rel_diff((fp - fm) / (2 * h), ju)
    f = host(op.apply_residual(cu(u)))  # restore the linearization state
    check("jacobian-fd", err < 1e-6, "relative error " + _fd(err))

    du = np.where(mask, 0.0, random_field(n, 33, 1.0))
    dpsi = (op.total_strain_energy(cu(u + h * du)) - op.total_strain_energy(cu(u - h * du))) / (2 * h)
    load = prob.load if prob.load is not None else np.zeros(n)
    fint_du = float(f @ du) + 1.0 * float(np.asarray(load) @ du)
    err = abs(fint_du - dpsi) / max(1.0, abs(dpsi))
    check("energy-gradient", err < 1e-6, "relative error " + _fd(err))

    xs, ys = random_field(n, 34, 1.0), random_field(n, 35, 1.0)
    g1 = float(host(op.apply_jacobian(cu(xs))) @ ys)
    g2 = float(xs @ host(op.apply_jacobian(cu(ys))))
    err = abs(g1 - g2) / max(1.0, abs(g1))
    check("jacobian-symmetry", err < 1e-11, "inner product gap " + _fd(err))

    A = AssembledOperator(op)
    A.numeric()
    xs = random_field(n, 36, 1.0)
    err = rel_diff(host(A.matvec(cu(xs))), host(op.apply_jacobian(cu(xs))))
    check("assembled-equivalence", err < 1e-12, "relative difference " + _fd(err))
    rp, cols, vals = A.csr()
    rows = np.repeat(np.arange(n), np.diff(rp))
    dcsr = np.zeros(n)
    dcsr[rows[rows == cols]] = vals[rows == cols]
    dd = rel_diff(host(op.extract_diagonal()), dcsr)
    check("diagonal-equivalence", dd < 1e-12, "relative difference " + _fd(dd))

    # Galerkin coarse identity and prolongation adjoint on the hierarchy.
    mg = prob.hierarchy
    mg.setup_numeric()
    fine = mg.num_levels() - 1
    nc = mg.level_size(fine - 1)
    xc = random_field(nc, 37, 1.0)
    pxc = mg.prolong(fine - 1, cu(xc))
    ral = host(mg.restrict_to(fine - 1, op.apply_jacobian(pxc)))
    amf = host(mg.level_operator(fine - 1).apply_jacobian(cu(xc)))
    from .hexmg import constraint_mask
    pc = next(p for p in range(1, 5)
              if 3 * np.prod([p * c + 1 for c in prob.cells]) == nc)  # coarse level order
    cm = np.asarray(constraint_mask(prob.cells, pc, ("-x",))[0]) != 0
    num = float(np.sum(((ral - amf) ** 2)[~cm]))
    den = float(np.sum((amf**2)[~cm]))
    err = float(np.sqrt(num / den))
    check("galerkin-identity", err < 1e-12, "relative difference " + _fd(err))
    yf = random_field(n, 38, 1.0)
    lhs = float(host(pxc) @ yf)
    rhs = float(xc @ host(mg.restrict_to(fine - 1, cu(yf))))
    aerr = abs(lhs - rhs) / max(1.0, abs(lhs))
    check("prolongation-adjoint", aerr < 1e-13, "inner product gap " + _fd(aerr))

    ok = STATE_SCALARS[0] == 17 and STATE_SCALARS[1] == 19 and STATE_SCALARS[2] == 26
    check("state-scalar-counts", ok, "current/native/tuned = 17/19/26")

    acc = _coo_to_csr([0, 0, -1, 1], [0, 0, 5, 1], [1.0, 2.0, 99.0, 4.0], 2)
    ok = len(acc) == 2 and acc[(0, 0)] == 3.0 and acc[(1, 1)] == 4.0
    check("coo-semantics", ok, "dup sum + negative discard")
    return res
