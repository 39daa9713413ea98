"""Dev helper (GPU box): locate partitioned-apply differences.
usage: python scripts/diag_partition.py px py pz"""
import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch, torch.multiprocessing as mp
from test_gpu_partitioned import _smooth_u, _free_port, _block, CELLS, EXT, TRACTION, rel

def run(rank, world, port, dims, out):
    import torch.distributed as dist
    from paper_2204_01722_b200.distributed import Communicator, PartitionedProblem
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, init_method=f"tcp://127.0.0.1:{port}")
    comm = Communicator(rank, world, dist, backend="gloo")
    pp = PartitionedProblem(comm, CELLS, dims, order=2, extents=EXT, fixed_faces=("-x",), traction_face="+x", traction=TRACTION)
    npd = tuple(2 * c + 1 for c in pp.cells); gnpd = tuple(2 * c + 1 for c in CELLS); node0 = tuple(2 * e for e in pp.e0)
    u = torch.from_numpy(_smooth_u(npd, node0, gnpd)).cuda()
    pp.residual(u)
    x = torch.from_numpy(_smooth_u(npd, node0, gnpd, 1.0)).cuda() * 3.0 + 1e-3
    yl = pp.op.apply_jacobian(x).cpu().numpy()
    y = pp.apply(x).cpu().numpy()
    np.savez(os.path.join(out, f"r{rank}.npz"), y=y, yl=yl, mask=pp.prob.mask, meta=np.array(list(npd) + list(node0)))
    dist.barrier(); dist.destroy_process_group()

if __name__ == "__main__":
    dims = tuple(int(a) for a in sys.argv[1:4]); world = dims[0] * dims[1] * dims[2]
    from paper_2204_01722_b200.hexmg import FemProblem
    prob = FemProblem(extents=EXT, cells=CELLS, order=2, fixed_faces=("-x",), traction_face="+x", traction=TRACTION, geometry="box")
    gnpd = tuple(2 * c + 1 for c in CELLS)
    prob.op.apply_residual(torch.from_numpy(_smooth_u(gnpd, (0, 0, 0), gnpd)).cuda())
    xg = torch.from_numpy(_smooth_u(gnpd, (0, 0, 0), gnpd, 1.0)).cuda() * 3.0 + 1e-3
    yg = prob.op.apply_jacobian(xg).cpu().numpy(); mg = prob.mask
    out = "/tmp/diagp"; os.makedirs(out, exist_ok=True)
    port = _free_port(); ctx = mp.get_context("spawn")
    ps = [ctx.Process(target=run, args=(r, world, port, dims, out)) for r in range(world)]
    [p.start() for p in ps]; [p.join() for p in ps]
    acc = np.zeros(gnpd[::-1] + (3,))
    for r in range(world):
        d = np.load(f"{out}/r{r}.npz"); npd = tuple(d["meta"][:3]); n0 = tuple(d["meta"][3:])
        yl = d["yl"].reshape(npd[2], npd[1], npd[0], 3).copy()
        m = d["mask"].reshape(yl.shape) != 0
        yl[m] = 0.0
        acc[n0[2]:n0[2]+npd[2], n0[1]:n0[1]+npd[1], n0[0]:n0[0]+npd[0]] += yl
        yb = _block(yg, gnpd, npd, n0).reshape(npd[2], npd[1], npd[0], 3)
        dd = np.abs(d["y"].reshape(yb.shape) - yb)
        bad = np.argwhere(dd > 1e-12 * np.abs(yg).max())
        print("rank", r, "npd", npd, "node0", n0, "rel", rel(d["y"], yb.ravel()), "nbad", len(bad), "first bad (z,y,x,c)", bad[:5].tolist())
    accf = acc.reshape(-1); gm = mg != 0
    print("assembled-from-locals vs global (unconstrained)", rel(accf[~gm], yg[~gm]))
