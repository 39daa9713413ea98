"""One coarse solve under an NVTX range (for ncu --nvtx-include 'csolve/')."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem
order, n = int(sys.argv[1]), int(sys.argv[2])
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",))
N = prob.size()
prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
mg = prob.hierarchy
mg.setup_numeric()
xk = torch.sin(torch.arange(mg.level_size(0), dtype=torch.float64, device="cuda"))
mg.coarse_solve(xk); torch.cuda.synchronize()
torch.cuda.nvtx.range_push("csolve")
mg.coarse_solve(xk); torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
xf = torch.sin(torch.arange(mg.level_size(1), dtype=torch.float64, device="cuda"))
torch.cuda.nvtx.range_push("restrict")
mg.restrict_to(0, xf); torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
