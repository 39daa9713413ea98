"""Fused residual vs the two-pass element path (variant 1): time, f and
exported state agreement.  usage: python scripts/res_time.py [order:cells,...]"""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2204_01722_b200.hexmg import FemProblem

cases = [tuple(map(int, c.split(":"))) for c in (sys.argv[1] if len(sys.argv) > 1 else "2:64,3:43,4:32").split(",")]
geo = sys.argv[2] if len(sys.argv) > 2 else "box"
for order, n in cases:
    prob = FemProblem(extents=(1, 1, 1), cells=(n, n, n), order=order, fixed_faces=("-x",),
                      traction_face="+x", traction=(0, 0, -0.02),
                      geometry="box" if geo == "box" else True)
    N = prob.size()
    gn = order * n + 1
    idx = torch.arange(N // 3, device="cuda", dtype=torch.float64)
    X = (idx % gn) / (gn - 1); Y = ((idx // gn) % gn) / (gn - 1); Z = (idx // (gn * gn)) / (gn - 1)
    sn = torch.sin(np.pi * X / 2) * torch.sin(np.pi * Y) * torch.sin(np.pi * Z)
    u = torch.stack([-0.05 * X + 0.02 * sn, 0.03 * sn, 0.01 * X * X], 1).reshape(-1).contiguous()
    u[torch.from_numpy(prob.mask).cuda() != 0] = 0.0
    out = {}
    for v in (1, 0):
        prob.op.set_variant(v)
        f = prob.op.apply_residual(u)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            prob.op.apply_residual(u, f)
        b.record(); torch.cuda.synchronize()
        st = prob.op.export_state(prob.num_elements, prob.nq) if n <= 48 else None
        out[v] = (a.elapsed_time(b) / 10, f.clone(), st)
    rel = float(torch.linalg.norm(out[0][1] - out[1][1]) / torch.linalg.norm(out[1][1]))
    srel = None
    if out[0][2] is not None:
        srel = float(np.abs(out[0][2] - out[1][2]).max() / np.abs(out[1][2]).max())
    print(json.dumps(dict(case=f"Q{order} {n}^3", geometry=geo, two_pass_ms=out[1][0], fused_ms=out[0][0],
                          f_rel=rel, state_maxrel=srel)), flush=True)
    del prob; torch.cuda.empty_cache()
