"""p-MG PCG solve timing (dev helper): python scripts/time_pmg.py order cells [mode] [rtol]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2204_01722_b200.hexmg import FemProblem, cg_solve
order = int(sys.argv[1]); n = int(sys.argv[2]); mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
rtol = float(sys.argv[4]) if len(sys.argv) > 4 else 1e-8
t0 = time.perf_counter()
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",), traction_face="+x", traction=(0, 0, -0.02))
N = prob.size()
f = prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
mg = prob.hierarchy; mg.set_coarse_mode(mode)
torch.cuda.synchronize(); t1 = time.perf_counter()
mg.setup_numeric(); torch.cuda.synchronize(); t2 = time.perf_counter()
r = cg_solve(prob.op, -f, rtol=rtol, precond="mg", mg=mg); torch.cuda.synchronize(); t3 = time.perf_counter()
b = -f; t4 = time.perf_counter(); x = mg.coarse_solve(torch.ones(mg.level_size(0), dtype=torch.float64, device="cuda")); torch.cuda.synchronize(); t5 = time.perf_counter()
print(f"Q{order} {n}^3 N={N} coarse={mg.level_size(0)} mode={mode} build {t1-t0:.2f}s setup {t2-t1:.3f}s solve {t3-t2:.3f}s its {r['iterations']} cond {r['eig_max']/r['eig_min']:.3f} coarse_solve {1e3*(t5-t4):.2f}ms", flush=True)
