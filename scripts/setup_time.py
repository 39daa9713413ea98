"""Exact-mode p-MG numeric setup timing (dev helper): second setup_numeric of
Q2 64^3 / Q3 43^3 / Q4 32^3 (the first includes the symbolic analysis), and
the PCG iteration count to 1e-8 after it."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem, cg_solve
cases = [(2, 64), (3, 43), (4, 32)] if len(sys.argv) < 2 else [tuple(map(int, c.split(":"))) for c in sys.argv[1].split(",")]
for order, n in cases:
    prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",),
                      traction_face="+x", traction=(0, 0, -0.02))
    f = prob.op.apply_residual(torch.zeros(prob.size(), dtype=torch.float64, device="cuda"))
    mg = prob.hierarchy; mg.set_coarse_mode("auto")
    mg.setup_numeric(); torch.cuda.synchronize()
    ts = []
    for _ in range(2):
        t0 = time.perf_counter(); mg.setup_numeric(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    r = cg_solve(prob.op, -f, rtol=1e-8, precond="mg", mg=mg)
    b = torch.sin(torch.arange(mg.level_size(0), dtype=torch.float64, device="cuda"))
    mg.coarse_solve(b); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10): mg.coarse_solve(b)
    torch.cuda.synchronize(); cs = (time.perf_counter() - t0) / 10
    print("RESULT", json.dumps({"case": f"Q{order} {n}^3", "setup_ms": [round(1e3 * t, 1) for t in ts],
                                "pcg_its": r["iterations"], "coarse_solve_ms": round(1e3 * cs, 2)}), flush=True)
