"""p-MG timing breakdown (dev helper, GPU box): setup, V-cycle pieces, PCG.
usage: python scripts/pmg_breakdown.py order cells [mode]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2204_01722_b200.hexmg import FemProblem, cg_solve

order, n = int(sys.argv[1]), int(sys.argv[2])
mode = sys.argv[3] if len(sys.argv) > 3 else "auto"
ev = lambda: torch.cuda.Event(enable_timing=True)
def timed(f, reps=3):
    f(); torch.cuda.synchronize()
    a, b = ev(), ev(); a.record()
    for _ in range(reps): f()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
t0 = time.perf_counter()
prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",),
                  traction_face="+x", traction=(0, 0, -0.02))
N = prob.size()
f = prob.op.apply_residual(torch.zeros(N, dtype=torch.float64, device="cuda"))
mg = prob.hierarchy; mg.set_coarse_mode(mode)
torch.cuda.synchronize(); t1 = time.perf_counter()
mg.setup_numeric(); torch.cuda.synchronize(); t2 = time.perf_counter()
setup2 = timed(mg.setup_numeric, 1)
L = mg.num_levels()
print(f"Q{order} {n}^3 N={N} levels={[mg.level_size(k) for k in range(L)]} build {t1-t0:.2f}s "
      f"setup(first) {1e3*(t2-t1):.1f} ms setup(again) {setup2:.1f} ms", flush=True)
b = -f
print(f"  v-cycle {timed(lambda: mg.v_cycle(b)):.2f} ms", flush=True)
for k in range(L):
    opk = mg.level_operator(k)
    xk = torch.sin(torch.arange(mg.level_size(k), dtype=torch.float64, device="cuda"))
    yk = torch.empty_like(xk)
    line = f"  level {k} n={mg.level_size(k)} apply {timed(lambda: opk.apply_jacobian(xk, yk), 10):.3f} ms"
    if k > 0:
        line += f" smooth {timed(lambda: mg.smooth(k, xk, yk), 5):.3f} ms"
        line += f" prolong {timed(lambda: mg.prolong(k - 1, torch.ones(mg.level_size(k-1), dtype=torch.float64, device='cuda')), 5):.3f} ms"
        line += f" restrict {timed(lambda: mg.restrict_to(k - 1, xk), 5):.3f} ms"
    else:
        line += f" coarse_solve {timed(lambda: mg.coarse_solve(xk), 5):.3f} ms"
    print(line, flush=True)
for rtol in (1e-3, 1e-8):
    r = {}
    def run():
        r.update(cg_solve(prob.op, b, rtol=rtol, precond="mg", mg=mg))
    ms = timed(run, 1)
    print(f"  PCG rtol {rtol:g}: {ms:.1f} ms, {r['iterations']} its, cond {r['eig_max']/r['eig_min']:.3f}", flush=True)
