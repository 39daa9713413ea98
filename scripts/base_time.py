"""Dense Cholesky+inverse base block timing (dev helper): one-front dense
CoarseCholesky on a random SPD lattice matrix, device-resident values,
factorize() wall time (assembly + dense_chol_inv + info read-back)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, scipy.sparse as sp, torch
from paper_2204_01722_b200.hexmg import CoarseCholesky

def lattice(npd, seed=7):
    nx, ny, nz = npd
    nodes = nx * ny * nz
    idx = np.arange(nodes).reshape(nz, ny, nx)
    rows, cols = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                a = idx[max(0, -dz):nz - max(0, dz), max(0, -dy):ny - max(0, dy), max(0, -dx):nx - max(0, dx)]
                b = idx[max(0, dz):nz - max(0, -dz), max(0, dy):ny - max(0, -dy), max(0, dx):nx - max(0, -dx)]
                rows.append(a.ravel()); cols.append(b.ravel())
    r = np.concatenate(rows); c = np.concatenate(cols); n = 3 * nodes
    R = (3 * r[:, None] + np.arange(3)[None, :]).repeat(3, 1).ravel()
    C = np.tile(3 * c[:, None] + np.arange(3)[None, :], (1, 3)).ravel()
    B = sp.csr_matrix((np.random.RandomState(seed).uniform(-1, 1, R.size), (R, C)), shape=(n, n))
    A = (B + B.T).tocsr()
    A = (A + sp.diags(np.asarray(abs(A).sum(1)).ravel() + 1.0)).tocsr(); A.sort_indices()
    return A

for npd in [(7, 3, 2), (8, 8, 4), (16, 8, 8), (16, 16, 16)]:
    A = lattice(npd)
    ch = CoarseCholesky(A.indptr, A.indices, npd, mode="dense")
    v = torch.from_numpy(A.data).cuda()
    ch.factorize(v); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20): ch.factorize(v)
    torch.cuda.synchronize()
    print(f"n={A.shape[0]:6d} dense factorize {1e3 * (time.perf_counter() - t0) / 20:8.3f} ms", flush=True)
