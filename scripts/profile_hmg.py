"""p-MG with the inexact coarse mode: setup + a few V-cycles (ncu captures of
the h-multigrid kernels).  usage: python scripts/profile_hmg.py [order] [cells] [mode]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem
order = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
mode = sys.argv[3] if len(sys.argv) > 3 else "hmg"
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",),
                  traction_face="+x", traction=(0, 0, -0.02))
f = prob.op.apply_residual(torch.zeros(prob.size(), dtype=torch.float64, device="cuda"))
mg = prob.hierarchy
mg.set_coarse_mode(mode)
mg.setup_numeric()
for _ in range(3):
    mg.v_cycle(-f)
torch.cuda.synchronize()
print("done")
