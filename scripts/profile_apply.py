"""Runs a few Jacobian applies at a BASELINE size for ncu captures.
usage: python scripts/profile_apply.py [order] [cells] [variant] [applies]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem
order = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
variant = int(sys.argv[3]) if len(sys.argv) > 3 else 0
applies = int(sys.argv[4]) if len(sys.argv) > 4 else 5
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order)
prob.op.set_variant(variant)
N = prob.size()
prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
x = torch.sin(0.7 * torch.arange(N, dtype=torch.float64, device="cuda")) * 1e-3
y = torch.empty_like(x)
for _ in range(applies):
    prob.op.apply_jacobian(x, y)
torch.cuda.synchronize()
print("done", N)
