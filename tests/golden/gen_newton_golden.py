"""Newton-with-load-continuation goldens from the UNMODIFIED reference
(oracle/_ref/libhexmg_ref.so: FemProblem::solve, problem.hpp:118-127,
newton_solve nonlinear.hpp:162-216, load_continuation :325-366).  Run in the
build container (needs /root/reference compiled into oracle/_ref):
    python tests/golden/gen_newton_golden.py
Writes tests/golden/newton.npz.  Config: Q2 bar, extents (2, 1, 1), cells
(4, 2, 2), fixed -x, traction on +x, E = 1, nu = 0.3; defaults of
config.hpp:55-61 (newton rtol 1e-8, atol 1e-10, max 50, linear rtol 1e-3)."""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref_lib as R  # noqa: E402

CASES = {
    # name: (traction, load_steps, line_search)
    "bend_ls0": ((0.0, 0.0, -0.02), 5, 0),
    "compress_ls0": ((-0.05, 0.0, 0.0), 5, 0),
    "bend_ls1": ((0.0, 0.0, -0.02), 5, 1),
    "compress1_ls0": ((-0.05, 0.0, 0.0), 1, 0),
}
out = {}
for name, (tr, steps, ls) in CASES.items():
    rp = R.RefProblem(extents=(2.0, 1.0, 1.0), cells=(4, 2, 2), order=2, fixed=("-x",),
                      traction_face="+x", traction=tr)
    r = rp.newton(load_steps=steps, line_search=bool(ls), linear_rtol=1e-3)
    out[f"{name}_u"] = r["u"]
    out[f"{name}_stats"] = np.array([r["newton_iterations"], r["cg_iterations"], r["final_fnorm"]])
    print(name, r["newton_iterations"], r["cg_iterations"], r["final_fnorm"])
# L-BFGS (config.hpp:15, memory 5, refresh 10) with the line search (its
# functor-copy defect makes it stop after one step per load step)
rp = R.RefProblem(extents=(2.0, 1.0, 1.0), cells=(4, 2, 2), order=2, fixed=("-x",),
                  traction_face="+x", traction=(-0.05, 0.0, 0.0))
r = rp.solve(load_steps=1, line_search=True, solver=1, memory=5, refresh=10)
out["lbfgs_compress1_u"] = r["u"]
out["lbfgs_compress1_stats"] = np.array([r["iterations"], r["cg_iterations"], r["final_fnorm"]])
print("lbfgs_compress1", r["iterations"], r["cg_iterations"], r["final_fnorm"])
np.savez(os.path.join(HERE, "newton.npz"), **out)
