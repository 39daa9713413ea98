"""The partitioned p-multigrid of the C++ library (hxg_mg_create_partitioned,
csrc/dist.cu + csrc/solver.cpp) against the single-process
library on the whole box.  World sizes 2, 3 (slabs along x) and 4 (2 x 2 x 1
blocks) run as processes sharing the one GPU, their communicator a table of
callbacks over a gloo process group (distributed.Communicator(backend="gloo"));
world 1 uses the built-in NCCL communicator.  NCCL with several ranks is the
only layer not exercised here (one GPU per box).

Checked per rank against the whole-box run restricted to the block:
Jacobian apply (the interface sums), residual, Chebyshev lambda_max per
level (global rough_seed slice: partition independent), p-MG PCG iterations
and solution (cg.hpp:81-134; the coarse level summed into the global Q1
matrix), and the Newton + load continuation solve (problem.hpp:118-127)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

EXT = (3.0, 1.0, 1.0)
CELLS = (12, 4, 4)
TRACTION = (0.0, 0.0, -0.02)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _smooth_u(npd, node0, gnpd, scale=0.2):
    """SURVEY.md §8(d) parity state on the global lattice, block slice."""
    nx, ny, nz = npd
    gz, gy, gx = np.meshgrid(np.arange(nz) + node0[2], np.arange(ny) + node0[1],
                             np.arange(nx) + node0[0], indexing="ij")
    X = EXT[0] * gx / (gnpd[0] - 1)
    Y = EXT[1] * gy / (gnpd[1] - 1)
    Z = EXT[2] * gz / (gnpd[2] - 1)
    s = np.sin(np.pi * X / 2) * np.sin(np.pi * Y) * np.sin(np.pi * Z)
    u = scale * np.stack([-0.05 * X + 0.02 * s, 0.03 * s, 0.01 * X**2], -1)
    u[gx == 0] = 0.0  # fixed -x
    return u.reshape(-1)


def _run(rank, world, port, dims, order, out_dir, cells=CELLS, mode="auto"):
    import torch.distributed as dist

    from paper_2204_01722_b200.distributed import Communicator, PartitionedProblem

    torch.cuda.set_device(0)
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world,
                                init_method=f"tcp://127.0.0.1:{port}")
    comm = Communicator(rank, world, dist if world > 1 else None,
                        backend="gloo" if world > 1 else "nccl")
    pp = PartitionedProblem(comm, cells, dims, order=order, extents=EXT, fixed_faces=("-x",),
                            traction_face="+x", traction=TRACTION)
    p = order
    npd = tuple(p * c + 1 for c in pp.cells)
    gnpd = tuple(p * c + 1 for c in cells)
    node0 = tuple(p * e for e in pp.e0)
    n = pp.size()
    res = {}
    u = torch.from_numpy(_smooth_u(npd, node0, gnpd)).cuda()
    res["f"] = pp.residual(u).cpu().numpy()
    x = torch.from_numpy(_smooth_u(npd, node0, gnpd, 1.0)).cuda() * 3.0 + 1e-3
    res["y"] = pp.apply(x).cpu().numpy()
    # linearised at u = 0 (b = -F(0)), p-MG PCG to 1e-8
    f0 = pp.residual(torch.zeros(n, dtype=torch.float64, device="cuda"))
    pp.set_coarse_mode(mode)
    pp.setup_numeric()
    res["lam"] = np.array([pp.lambda_max(k) for k in range(1, pp.levels)])
    r = pp.cg_solve(-f0, rtol=1e-8)
    res["its"] = np.array([r["iterations"]])
    res["x"] = r["x"].cpu().numpy()
    s = pp.solve(load_steps=2)
    res["newton"] = np.array([s["newton_iterations"], s["cg_iterations"]])
    res["u"] = s["u"].cpu().numpy()
    res["meta"] = np.array(list(npd) + list(node0))
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **res)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _whole_box(order, cells=CELLS, mode="auto"):
    from paper_2204_01722_b200.hexmg import FemProblem, cg_solve
    prob = FemProblem(extents=EXT, cells=cells, order=order, fixed_faces=("-x",),
                      traction_face="+x", traction=TRACTION, geometry="box")
    gnpd = tuple(order * c + 1 for c in cells)
    n = prob.size()
    out = {}
    u = torch.from_numpy(_smooth_u(gnpd, (0, 0, 0), gnpd)).cuda()
    out["f"] = prob.op.apply_residual(u).cpu().numpy()
    x = torch.from_numpy(_smooth_u(gnpd, (0, 0, 0), gnpd, 1.0)).cuda() * 3.0 + 1e-3
    out["y"] = prob.op.apply_jacobian(x).cpu().numpy()
    f0 = prob.op.apply_residual(torch.zeros(n, dtype=torch.float64, device="cuda"))
    mg = prob.hierarchy
    mg.set_coarse_mode(mode)
    mg.setup_numeric()
    out["lam"] = np.array([mg.lambda_max(k) for k in range(1, mg.num_levels())])
    r = cg_solve(prob.op, -f0, rtol=1e-8, precond="mg", mg=mg)
    out["its"], out["x"] = r["iterations"], r["x"].cpu().numpy()
    s = prob.solve(load_steps=2)
    out["newton"] = (s["newton_iterations"], s["cg_iterations"])
    out["u"] = s["u"].cpu().numpy()
    return out, gnpd


def _block(v, gnpd, npd, node0):
    g = v.reshape(gnpd[2], gnpd[1], gnpd[0], 3)
    return g[node0[2]:node0[2] + npd[2], node0[1]:node0[1] + npd[1],
             node0[0]:node0[0] + npd[0]].reshape(-1)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("world,dims,order", [(1, (1, 1, 1), 2), (2, (2, 1, 1), 2),
                                              (3, (3, 1, 1), 2), (4, (2, 2, 1), 2),
                                              (2, (2, 1, 1), 3)])
def test_partitioned_matches_whole_box(world, dims, order, tmp_path):
    _check_partitioned(world, dims, order, tmp_path, CELLS, "auto")


@pytest.mark.parametrize("world,dims", [(1, (1, 1, 1)), (2, (2, 1, 1)), (4, (2, 2, 1)), (8, (2, 2, 2))])
def test_partitioned_inexact_coarse_matches_whole_box(world, dims, tmp_path):
    """The inexact coarse mode distributed with the hierarchy (csrc/hcoarse.cu):
    h-levels on the blocks (32 x 16 x 16 Q2: the Q1 level and two Galerkin
    levels), replicated dense bottom -- the same lambda_max, iterations and
    solutions as the single-process h-multigrid."""
    _check_partitioned(world, dims, 2, tmp_path, (32, 16, 16), "hmg")


def _check_partitioned(world, dims, order, tmp_path, cells, mode):
    import torch.multiprocessing as mp
    ref, gnpd = _whole_box(order, cells, mode)
    port = _free_port()
    if world == 1:
        _run(0, 1, port, dims, order, str(tmp_path), cells, mode)
    else:
        ctx = mp.get_context("spawn")
        procs = [ctx.Process(target=_run, args=(r, world, port, dims, order, str(tmp_path), cells, mode))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(600)
        assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    for r in range(world):
        d = np.load(tmp_path / f"rank{r}.npz")
        npd, node0 = tuple(d["meta"][:3]), tuple(d["meta"][3:])
        assert rel(d["y"], _block(ref["y"], gnpd, npd, node0)) < 1e-13
        assert rel(d["f"], _block(ref["f"], gnpd, npd, node0)) < 1e-12
        assert np.allclose(d["lam"], ref["lam"], rtol=1e-10, atol=0)
        assert abs(int(d["its"][0]) - ref["its"]) <= 1
        assert rel(d["x"], _block(ref["x"], gnpd, npd, node0)) < 1e-7
        assert tuple(d["newton"]) == ref["newton"] or abs(int(d["newton"][1]) - ref["newton"][1]) <= 2
        assert rel(d["u"], _block(ref["u"], gnpd, npd, node0)) < 1e-6
