"""End-to-end (host buffers) apply: PCIe bandwidth per direction and
concurrent, and hxg_op_apply_jacobian_host for several chunk counts.
usage: HXG_HOST_CHUNKS=<c> python scripts/e2e_probe.py"""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem

prob = FemProblem(extents=(1, 1, 1), cells=(64, 64, 64), order=2, fixed_faces=("-x",), geometry="box")
N = prob.size()
prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
x = 1e-3 * torch.sin(0.7 * torch.arange(N, dtype=torch.float64, device="cuda"))
xh = x.cpu().pin_memory(); yh = torch.empty_like(xh).pin_memory()
d1, d2 = torch.empty_like(x), torch.empty_like(x)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, n=20):
    f(); torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - a) / n
h2d = t(lambda: d1.copy_(xh, non_blocking=True))
d2h = t(lambda: yh.copy_(d1, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d1.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2): yh.copy_(d2, non_blocking=True)
bo = t(both)
xn, yn = xh.numpy(), yh.numpy()
app = t(lambda: prob.op.apply_jacobian_host(xn, yn), 30)
print(json.dumps({"chunks": os.environ.get("HXG_HOST_CHUNKS", "default"), "bytes": 8 * N,
                  "h2d_GBs": 8 * N / h2d / 1e9, "d2h_GBs": 8 * N / d2h / 1e9,
                  "both_ms": bo * 1e3, "e2e_ms": app * 1e3, "e2e_GDoFs": N / app / 1e9}), flush=True)
