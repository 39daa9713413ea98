import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2204_01722_b200.hexmg import FemProblem
g = np.load('tests/golden/q2_bar.npz')
def rel(a,b): return np.linalg.norm(a-b)/np.linalg.norm(b)
for trial in range(4):
    prob = FemProblem(extents=(2.0, 1.0, 1.0), cells=(4,2,2), order=2, fixed_faces=("-x",), traction_face="+x", traction=(0.0, 0.0, -0.02))
    f = prob.op.apply_residual(torch.from_numpy(g['u']).cuda())
    print('res', rel(f.cpu().numpy(), g['f']))
    if trial == 1: torch.cuda.synchronize()
    xt = torch.from_numpy(g['x']).cuda()
    y1 = prob.op.apply_jacobian(xt).cpu().numpy()
    y2 = prob.op.apply_jacobian(torch.from_numpy(g['x']).cuda()).cpu().numpy()
    y3 = prob.op.apply_jacobian(xt).cpu().numpy()
    print(trial, 'kept', rel(y1, g['jx']), 'temp', rel(y2, g['jx']), 'kept again', rel(y3, g['jx']))
    d = np.abs(y1-g['jx']); i = np.argsort(-d)[:8]; print('  worst idx', i, d[i])
