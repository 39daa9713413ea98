"""One numeric setup under an NVTX range (ncu --nvtx-include 'setup/')."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem
order, n = int(sys.argv[1]), int(sys.argv[2])
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",))
prob.op.apply_residual(torch.zeros(prob.size(), dtype=torch.float64, device="cuda"))
mg = prob.hierarchy
mg.setup_numeric(); torch.cuda.synchronize()
torch.cuda.nvtx.range_push("setup")
mg.setup_numeric(); torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
