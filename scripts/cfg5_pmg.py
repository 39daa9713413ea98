"""BASELINE configs[4] per-GPU size: Q2 160^3 cube (99.2 M DoF), p-MG solve
with the inexact coarse mode (an exact factorisation of the 12.5 M-DoF Q1
level is infeasible); device-timed residual, setup_numeric, PCG to 1e-8.
usage: python scripts/cfg5_pmg.py [cells] [order]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem, cg_solve

n = int(sys.argv[1]) if len(sys.argv) > 1 else 160
order = int(sys.argv[2]) if len(sys.argv) > 2 else 2
t0 = time.perf_counter()
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",),
                  traction_face="+x", traction=(0, 0, -0.02), geometry="box")
N = prob.size()
z = torch.zeros(N, dtype=torch.float64, device="cuda")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
f = prob.op.apply_residual(z)
mg = prob.hierarchy
mg.set_coarse_mode("hmg")
t1 = time.perf_counter()
mg.setup_numeric()  # symbolic (patterns, host) + numeric
torch.cuda.synchronize()
t2 = time.perf_counter()
ev[0].record()
f = prob.op.apply_residual(z)
ev[1].record()
mg.setup_numeric()
ev[2].record()
r = cg_solve(prob.op, -f, rtol=1e-8, precond="mg", mg=mg)
ev[3].record()
torch.cuda.synchronize()
print(json.dumps({"config": f"Q{order} {n}^3 cube, fixed -x, traction (0,0,-0.02) on +x, u = 0, inexact coarse",
                  "dofs": N, "levels": [mg.level_size(k) for k in range(mg.num_levels())],
                  "h_levels": mg.hmg_levels(), "build_s": t1 - t0, "first_setup_s": t2 - t1,
                  "residual_ms": ev[0].elapsed_time(ev[1]), "setup_numeric_ms": ev[1].elapsed_time(ev[2]),
                  "pcg_rtol1e-8_ms": ev[2].elapsed_time(ev[3]), "pcg_iterations": r["iterations"],
                  "converged": r["converged"], "condition": r["eig_max"] / r["eig_min"],
                  "peak_mem_GB": torch.cuda.max_memory_allocated() / 1e9}), flush=True)
