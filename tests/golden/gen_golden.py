"""Generate the golden parity fixtures in tests/golden/ from the reference itself.

Runs the UNMODIFIED reference headers compiled into oracle/_ref/libhexmg_ref.so
(oracle/Makefile; needs /root/reference, i.e. this container only) and stores
small .npz fixtures that travel with the repo.  Re-run with
    python tests/golden/gen_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import ref_lib as R  # noqa: E402


def parity_state(rp, scale):
    """Smooth tau != 0 linearization point (SURVEY.md §8(d) parity state)."""
    X = rp.coords()
    ext = rp.extents
    s = (np.sin(np.pi * X[:, 0] / ext[0]) * np.sin(np.pi * X[:, 1] / ext[1])
         * np.sin(np.pi * X[:, 2] / ext[2]))
    u = scale * np.stack([-0.05 * X[:, 0] + 0.02 * s, 0.03 * s, 0.01 * X[:, 0] ** 2], 1).ravel()
    m, _ = rp.constraints()
    u[m != 0] = 0.0
    return u


def gen_basis():
    out = {}
    for p, q in [(1, 2), (2, 3), (3, 4), (4, 5), (1, 3), (1, 4), (1, 5), (2, 4), (2, 5)]:
        b = R.basis(p, q)
        for k, v in b.items():
            out[f"p{p}q{q}_{k}"] = v
    np.savez_compressed(os.path.join(HERE, "basis.npz"), **out)


def gen_cfg1():
    """cfg1: linear elasticity (Neo-Hookean at u = 0), Q1 unit cube 8^3,
    Jacobi-CG (BASELINE.json configs[0])."""
    rp = R.RefProblem(extents=(1, 1, 1), cells=(8, 8, 8), order=1, fixed=("-x",),
                      traction_face="+x", traction=(0, 0, -0.02))
    u = rp.impose_dirichlet(np.zeros(rp.n))
    f = rp.apply_residual(u)
    out = dict(f0=f, diag=rp.extract_diagonal())
    for tag, rtol in (("1e-3", 1e-3), ("1e-8", 1e-8)):
        r = rp.cg(-f, "jacobi", rtol, 5000)
        out[f"x_{tag}"] = r["x"]
        out[f"its_{tag}"] = np.array(r["iterations"])
        out[f"cond_{tag}"] = np.array(r["eig_max"] / r["eig_min"])
    np.savez_compressed(os.path.join(HERE, "cfg1_q1_8.npz"), **out)


def gen_operator(order, cells, extents, scale, name):
    rp = R.RefProblem(extents=extents, cells=cells, order=order, fixed=("-x",),
                      traction_face="+x", traction=(0, 0, -0.02))
    u = parity_state(rp, scale)
    f = rp.apply_residual(u)
    n = rp.n
    x = 1e-3 * np.sin(0.7 * np.arange(n))
    rng = np.random.RandomState(7)
    out = dict(u=u, f=f, state=rp.state(), x=x, jx=rp.apply_jacobian(x),
               diag=rp.extract_diagonal(), load=rp.external_load())
    rp.mg_setup()
    L = rp.num_levels
    for k in range(L - 1):
        xc = rng.uniform(-1, 1, rp.level_size(k))
        xf = rng.uniform(-1, 1, rp.level_size(k + 1))
        out[f"P{k}_xc"], out[f"P{k}_pxc"] = xc, rp.prolong(k, xc)
        out[f"P{k}_xf"], out[f"P{k}_rxf"] = xf, rp.restrict(k, xf)
    for k in range(1, L):
        out[f"lam{k}"] = np.array(rp.lambda_max(k))
        out[f"jx_level{k}"] = rp.apply_jacobian(rng.uniform(-1, 1, rp.level_size(k)) * 0 + np.cos(0.3 * np.arange(rp.level_size(k))), k)
        out[f"diag_level{k}"] = rp.extract_diagonal(k)
    rc = rp.coarse_csr()
    out["coarse_rowptr"], out["coarse_cols"], out["coarse_vals"] = rc
    b = -f
    out["vcycle_b"] = b
    out["vcycle_x"] = rp.vcycle(b)
    for tag, rtol in (("1e-3", 1e-3), ("1e-8", 1e-8)):
        r = rp.cg(b, "mg", rtol, 500)
        out[f"mgcg_x_{tag}"] = r["x"]
        out[f"mgcg_its_{tag}"] = np.array(r["iterations"])
        out[f"mgcg_cond_{tag}"] = np.array(r["eig_max"] / r["eig_min"])
    out["meta"] = np.array([order, *cells, *extents, scale])
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


STORAGES = {1: "initial-native", 2: "initial-tuned", 3: "initial-ad"}


def gen_storage():
    """JacobianStorage variants (material.hpp:66-78, paper Table III):
    residual, state, Jacobian apply, diagonal and the p-MG PCG of the
    reference with each initial-configuration storage."""
    out = {}
    for order, cells, ext, name in ((2, (4, 2, 2), (2.0, 1.0, 1.0), "q2"),
                                    (3, (2, 2, 2), (1.0, 1.0, 1.0), "q3")):
        for st in STORAGES:
            rp = R.RefProblem(extents=ext, cells=cells, order=order, fixed=("-x",),
                              traction_face="+x", traction=(0, 0, -0.02), storage=st)
            u = parity_state(rp, 0.2)
            k = f"{name}_s{st}_"
            out[k + "u"], out[k + "f"] = u, rp.apply_residual(u)
            out[k + "state"] = rp.state()
            x = 1e-3 * np.sin(0.7 * np.arange(rp.n))
            out[k + "x"], out[k + "jx"] = x, rp.apply_jacobian(x)
            out[k + "diag"] = rp.extract_diagonal()
            out[k + "bytes_per_dof"] = np.array(rp.stored_bytes_per_dof())
            rp.mg_setup()
            b = -out[k + "f"]
            out[k + "vcycle_x"] = rp.vcycle(b)
            r = rp.cg(b, "mg", 1e-8, 500)
            out[k + "mgcg_x"], out[k + "mgcg_its"] = r["x"], np.array(r["iterations"])
            out[k + "meta"] = np.array([order, *cells, *ext])
    np.savez_compressed(os.path.join(HERE, "storage.npz"), **out)


def gen_verify():
    res = R.verify(threads=1)
    bad = R.verify(threads=1, perturbation=1e-3)
    names = sorted(res)
    np.savez_compressed(os.path.join(HERE, "verify.npz"), names=np.array(names),
                        passed=np.array([res[k][0] for k in names]),
                        passed_perturbed=np.array([bad[k][0] for k in names]))


if __name__ == "__main__":
    gen_basis()
    gen_cfg1()
    gen_operator(2, (4, 2, 2), (2.0, 1.0, 1.0), 0.2, "q2_bar")
    gen_operator(3, (2, 2, 2), (1.0, 1.0, 1.0), 0.2, "q3_cube")
    gen_operator(4, (2, 2, 1), (1.0, 1.0, 1.0), 0.2, "q4_cube")
    gen_operator(1, (4, 2, 2), (2.0, 1.0, 1.0), 0.2, "q1_bar")
    gen_verify()
    gen_storage()
    print("ok")
