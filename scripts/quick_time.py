"""Quick device timing of the Jacobian apply at BASELINE sizes (dev helper)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem

for order, n in [(2, 64), (3, 43), (4, 32), (1, 64)]:
    t0 = time.time()
    prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order)
    N = prob.size()
    prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
    x = torch.sin(0.7 * torch.arange(N, dtype=torch.float64, device="cuda")) * 1e-3
    y = torch.empty_like(x)
    bpd = prob.op.stored_bytes_per_dof()
    for v in (0, 1):
        prob.op.set_variant(v)
        ms = prob.op.time_jacobian(x, y, 3, 20) / 20
        gdofs = N / ms / 1e6
        print(f"Q{order} {n}^3 N={N} variant={v} {ms*1e3:.1f} us/apply {gdofs:.2f} GDoF/s "
              f"{gdofs*bpd:.0f} GB/s (model {bpd:.1f} B/DoF) setup {time.time()-t0:.1f}s", flush=True)
