"""One p-MG Newton-Krylov step at a given size (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem, cg_solve
order = int(sys.argv[1]); n = int(sys.argv[2])
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",), traction_face="+x", traction=(0, 0, -0.02))
u = torch.zeros(prob.size(), dtype=torch.float64, device="cuda")
f = prob.op.apply_residual(u)
mg = prob.hierarchy
mg.setup_numeric()
r = cg_solve(prob.op, -f, rtol=1e-3, precond="mg", mg=mg)
torch.cuda.synchronize()
print("its", r["iterations"])
