"""A few fused residual applies at a BASELINE size for ncu captures.
usage: python scripts/profile_residual.py [order] [cells] [applies]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem
order = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
applies = int(sys.argv[3]) if len(sys.argv) > 3 else 4
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",))
u = 1e-3 * torch.sin(1e-3 * torch.arange(prob.size(), dtype=torch.float64, device="cuda"))
for _ in range(applies):
    prob.op.apply_residual(u)
torch.cuda.synchronize()
print("done")
