"""Dev helper (GPU box): per-scalar state / residual differences against the
compiled reference.  usage: python scripts/diag_state.py order n geometry(box|host)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import ref_lib as R
from paper_2204_01722_b200.hexmg import FemProblem
order, n, geo = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
ref = R.RefProblem(extents=(1, 1, 1), cells=(n,) * 3, order=order, fixed=("-x",), threads=os.cpu_count())
prob = FemProblem(extents=(1, 1, 1), cells=(n,) * 3, order=order, fixed_faces=("-x",),
                  geometry="box" if geo == "box" else True)
X = ref.coords(); mask = prob.mask
s = np.sin(np.pi * X[:, 0] / 2) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])
u = np.stack([-0.05 * X[:, 0] + 0.02 * s, 0.03 * s, 0.01 * X[:, 0] ** 2], 1).ravel(); u[mask != 0] = 0
f_ref = ref.apply_residual(u)
f = prob.op.apply_residual(torch.from_numpy(u).cuda()).cpu().numpy()
print("residual rel", np.linalg.norm(f - f_ref) / np.linalg.norm(f_ref), "max abs", np.abs(f - f_ref).max(),
      "at", np.argmax(np.abs(f - f_ref)), "of", f.size)
st_ref = ref.state(); st = prob.op.export_state(prob.num_elements, prob.nq)
d = np.abs(st - st_ref)
for k in range(st.shape[2]):
    e, q = np.unravel_index(np.argmax(d[:, :, k]), d.shape[:2])
    print(f"scalar {k:2d} maxdiff {d[:, :, k].max():.3e} scale {np.abs(st_ref[:, :, k]).max():.3e} "
          f"at e={e} (ex,ey,ez)=({e % n},{e // n % n},{e // n // n}) q={q} ours {st[e, q, k]!r} ref {st_ref[e, q, k]!r}")
