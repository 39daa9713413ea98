"""Exact (nested-dissection) vs inexact (h-multigrid) coarse mode: p-MG
setup_numeric, V-cycle and PCG (rtol 1e-3 / 1e-8) device times and
iterations.  usage: python scripts/hmg_eval.py [order:cells,...] [modes]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2204_01722_b200.hexmg import FemProblem, cg_solve

cases = [tuple(map(int, c.split(":"))) for c in (sys.argv[1] if len(sys.argv) > 1 else "2:16,2:64,3:43,4:32").split(",")]
modes = (sys.argv[2] if len(sys.argv) > 2 else "auto,hmg").split(",")


def timed(f, reps=1):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    for _ in range(reps):
        out = f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps, out


for order, n in cases:
    prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",),
                      traction_face="+x", traction=(0, 0, -0.02))
    N = prob.size()
    f = prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
    mg = prob.hierarchy
    xs = {}
    for mode in modes:
        mg.set_coarse_mode(mode)
        mg.setup_numeric()  # symbolic + first numeric
        t_setup, _ = timed(mg.setup_numeric)
        t_v, _ = timed(lambda: mg.v_cycle(-f), 5)
        t3, r3 = timed(lambda: cg_solve(prob.op, -f, rtol=1e-3, precond="mg", mg=mg))
        t8, r8 = timed(lambda: cg_solve(prob.op, -f, rtol=1e-8, precond="mg", mg=mg))
        xs[mode] = r8["x"]
        rec = dict(case=f"Q{order} {n}^3", N=N, mode=mode, setup_ms=t_setup, vcycle_ms=t_v,
                   pcg3_ms=t3, its3=r3["iterations"], pcg8_ms=t8, its8=r8["iterations"],
                   cond=r8["eig_max"] / r8["eig_min"], conv=r8["converged"])
        if mode != modes[0]:
            x0 = xs[modes[0]]
            rec["rel_vs_" + modes[0]] = float(torch.linalg.norm(r8["x"] - x0) / torch.linalg.norm(x0))
        print(json.dumps(rec), flush=True)
    del mg, prob
    torch.cuda.empty_cache()
