import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2204_01722_b200 import capi
from paper_2204_01722_b200.hexmg import FemProblem
order = int(sys.argv[1]) if len(sys.argv) > 1 else 2; n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order)
N = prob.size(); prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
x = torch.sin(0.7 * torch.arange(N, dtype=torch.float64, device="cuda")); y = torch.empty_like(x)
L = capi.lib(); buf = (ctypes.c_ulonglong * 10)()
prob.op.apply_jacobian(x, y); L.hxg_debug_phase_cycles(buf, 1)
for _ in range(5): prob.op.apply_jacobian(x, y)
L.hxg_debug_phase_cycles(buf, 1)
nb = prob.op.num_bricks() if hasattr(prob.op, 'num_bricks') else (n + 3) // 4 * ((n + 3) // 4) * ((n + 1) // 2)
v = np.array(list(buf), dtype=float) / 5 / nb
names = {0: "x block wait+mask", 1: "P1 (x,y passes)", 2: "P2 z pass + QF", 3: "Q1 z adjoint",
         4: "Q2 (y,x adjoint)", 5: "exp3", 8: "overlap-add+store"}
tot = v[:9].sum()
for i, c in enumerate(v[:9]):
    if c: print(f"{names.get(i, i)!s:20s} {c:8.0f} cycles/brick {100*c/tot:5.1f}%")
print("total", tot)
