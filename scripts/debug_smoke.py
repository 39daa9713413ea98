import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import hexmg_np as H
from paper_2204_01722_b200.hexmg import FemProblem
g = np.load('tests/golden/q2_bar.npz')
cells, order = (4, 2, 2), 2
prob = FemProblem(extents=(2.0, 1.0, 1.0), cells=cells, order=order, fixed_faces=("-x",), traction_face="+x", traction=(0.0, 0.0, -0.02))
ref = H.make_problem((2.0, 1.0, 1.0), cells, order, traction_face=1, traction=(0, 0, -0.02))
X = ref.mesh.coords
s = np.sin(np.pi * X[:, 0] / 2) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])
u = 0.2 * np.stack([-0.05 * X[:, 0] + 0.02 * s, 0.03 * s, 0.01 * X[:, 0] ** 2], 1).ravel()
u[ref.op.mask != 0] = 0.0
print('u vs golden', np.abs(u - g['u']).max())
f_ref = ref.op.apply_residual(u)
f = prob.op.apply_residual(torch.from_numpy(u).cuda()).cpu().numpy()
print('res', np.linalg.norm(f-f_ref)/np.linalg.norm(f_ref))
x = 1e-3 * np.sin(0.7 * np.arange(u.size))
print('x vs golden', np.abs(x-g['x']).max())
y_ref = ref.op.apply_jacobian(x)
print('yref vs golden', np.linalg.norm(y_ref-g['jx'])/np.linalg.norm(g['jx']))
for trial in range(3):
    xt = torch.from_numpy(x).cuda()
    y = prob.op.apply_jacobian(xt).cpu().numpy()
    print('jac', trial, np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref))
st = prob.op.export_state(prob.num_elements, prob.nq)
print('state', np.abs(st - ref.op.state).max())
y = prob.op.apply_jacobian(torch.from_numpy(x).cuda()).cpu().numpy()
print('jac after export', np.linalg.norm(y - y_ref) / np.linalg.norm(y_ref))
