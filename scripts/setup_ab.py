"""A/B of the p-MG numeric setup time across library variants (dev helper)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, torch, json
sys.path.insert(0, ROOT)
from paper_2204_01722_b200.hexmg import FemProblem
out = {}
for order, n in ((2, 64), (3, 43), (4, 32)):
    prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",))
    prob.op.apply_residual(torch.zeros(prob.size(), dtype=torch.float64, device="cuda"))
    mg = prob.hierarchy; mg.setup_numeric(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2): mg.setup_numeric()
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) / 2 * 1e3
    b = torch.sin(torch.arange(mg.level_size(0), dtype=torch.float64, device="cuda"))
    x0 = mg.coarse_solve(b); torch.cuda.synchronize()
    t1 = time.perf_counter()
    for _ in range(5): mg.coarse_solve(b)
    torch.cuda.synchronize()
    out[f"Q{order}"] = {"setup_ms": setup_ms, "solve_ms": (time.perf_counter() - t1) / 5 * 1e3,
                        "x": float(x0[:50].sum())}
    del mg, prob
print("RESULT", json.dumps(out))
'''
for lib in sys.argv[1:]:
    o = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT))],
                       env=dict(os.environ, HXG_LIBRARY=os.path.abspath(lib)), capture_output=True, text=True)
    line = [l for l in o.stdout.splitlines() if l.startswith("RESULT")]
    print(os.path.basename(lib), line[0][7:] if line else o.stderr[-400:], flush=True)
