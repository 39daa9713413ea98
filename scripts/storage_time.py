import torch, sys
sys.path.insert(0, '/root/repo')
from paper_2204_01722_b200.hexmg import FemProblem
for s in ("current", "initial-native", "initial-tuned", "initial-ad"):
    p = FemProblem(cells=(64,64,64), order=2, fixed_faces=("-x",), geometry="box", storage=s)
    n = p.size(); p.op.apply_residual(torch.zeros(n, dtype=torch.float64, device="cuda"))
    x = 1e-3*torch.sin(0.7*torch.arange(n, dtype=torch.float64, device="cuda")); y = torch.empty_like(x)
    res = {}
    for v in (0, 1):
        p.op.set_variant(v)
        for _ in range(3): p.op.apply_jacobian(x, y)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize(); e[0].record()
        for _ in range(20): p.op.apply_jacobian(x, y)
        e[1].record(); torch.cuda.synchronize()
        res[v] = e[0].elapsed_time(e[1]) / 20
        if v == 0: y0 = y.clone()
    rel = ((y - y0).norm() / y0.norm()).item()
    print(s, f"fused {res[0]:.3f} ms  two-pass {res[1]:.3f} ms  rel {rel:.2e}", flush=True)
    del p, x, y; torch.cuda.empty_cache()
