"""A/B of the coarse solve time across library variants (dev helper)."""
import os, subprocess, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, torch, json
sys.path.insert(0, ROOT)
from paper_2204_01722_b200.hexmg import FemProblem
prob = FemProblem(extents=(1, 1, 1), cells=(64, 64, 64), order=2, fixed_faces=("-x",))
prob.op.apply_residual(torch.zeros(prob.size(), dtype=torch.float64, device="cuda"))
mg = prob.hierarchy; mg.setup_numeric()
b = torch.sin(torch.arange(mg.level_size(0), dtype=torch.float64, device="cuda"))
x = mg.coarse_solve(b); torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
e[0].record()
for _ in range(10): mg.coarse_solve(b)
e[1].record(); torch.cuda.synchronize()
print("RESULT", json.dumps({"ms": e[0].elapsed_time(e[1]) / 10, "x0": float(x[:100].sum())}))
'''
for lib in sys.argv[1:]:
    out = subprocess.run([sys.executable, "-c", CHILD.replace("ROOT", repr(ROOT))],
                         env=dict(os.environ, HXG_LIBRARY=os.path.abspath(lib)), capture_output=True, text=True)
    line = [l for l in out.stdout.splitlines() if l.startswith("RESULT")]
    print(os.path.basename(lib), line[0][7:] if line else out.stderr[-400:], flush=True)
