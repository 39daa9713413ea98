"""A/B timing of library variants (dev helper, runs on the GPU box).
usage: python scripts/ab_time.py [--cases 2:64,3:43,4:32] [--rounds 2] lib1.so lib2.so ...
Each library runs in its own subprocess (HXG_LIBRARY); prints us/apply and
the relative difference of y against the first library's y."""
import argparse, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, os, json, numpy as np, torch
sys.path.insert(0, ROOT)
from paper_2204_01722_b200.hexmg import FemProblem
out = {}
for case in CASES:
    order, n = case
    prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",))
    N = prob.size()
    s = torch.arange(N, dtype=torch.float64, device="cuda")
    prob.op.apply_residual(1e-3 * torch.sin(1e-3 * s))  # tau != 0 state
    x = 1e-3 * torch.sin(0.7 * s)
    y = torch.empty_like(x)
    ms = prob.op.time_jacobian(x, y, 5, 50) / 50
    prob.op.apply_jacobian(x, y)
    y2 = torch.empty_like(x); prob.op.apply_jacobian(x, y2)
    np.save(f"/tmp/ab_{TAG}_{order}_{n}.npy", y.cpu().numpy())
    out[f"Q{order}_{n}"] = {"us": ms * 1e3, "N": N, "det": bool(torch.equal(y, y2))}
print("RESULT", json.dumps(out))
'''

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="2:64,3:43,4:32")
ap.add_argument("--rounds", type=int, default=2)
ap.add_argument("libs", nargs="+")
a = ap.parse_args()
cases = [tuple(map(int, c.split(":"))) for c in a.cases.split(",")]
import numpy as np
res = {}
for r in range(a.rounds):
    for i, libp in enumerate(a.libs):
        code = CHILD.replace("ROOT", repr(ROOT)).replace("CASES", repr(cases)).replace("TAG", str(i))
        env = dict(os.environ, HXG_LIBRARY=os.path.abspath(libp))
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
        line = [l for l in p.stdout.splitlines() if l.startswith("RESULT")]
        if not line:
            print(libp, "FAILED", p.stderr[-2000:], flush=True)
            continue
        d = json.loads(line[0][7:])
        for k, v in d.items():
            if i > 0:
                y0 = np.load(f"/tmp/ab_0_{k[1]}_{k.split('_')[1]}.npy")
                y1 = np.load(f"/tmp/ab_{i}_{k[1]}_{k.split('_')[1]}.npy")
                v["rel_vs_0"] = float(np.linalg.norm(y1 - y0) / np.linalg.norm(y0))
            res.setdefault((libp, k), []).append(v)
        print(r, os.path.basename(libp), json.dumps(d), flush=True)
print("SUMMARY (min us over rounds)")
for (libp, k), vs in sorted(res.items(), key=lambda kv: (kv[0][1], kv[0][0])):
    print(f"{k:10s} {min(v['us'] for v in vs):8.1f} us  det={all(v['det'] for v in vs)} "
          f"rel={vs[-1].get('rel_vs_0', 0):.2e}  {os.path.basename(libp)}")
