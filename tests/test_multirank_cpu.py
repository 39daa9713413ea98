"""World-size-2 CPU tests (gloo) of the multi-GPU host logic: slab partition,
interface-plane exchange and owned-entry dots.  Each rank
applies the oracle operator to its slab; after the exchange the slab result
must equal the global apply restricted to the slab, bitwise-identical on the
shared plane, and the distributed dot must equal the global one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hexmg_np as H
from dist_partition_model import exchange_faces, global_dot, owned_mask, slab_partition

GLOBAL_CELLS = (6, 2, 2)
EXT = (3.0, 1.0, 1.0)
ORDER = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _global_fields():
    P = H.make_problem(EXT, GLOBAL_CELLS, ORDER, fixed_faces=(0,))
    X = P.mesh.coords
    s = np.sin(np.pi * X[:, 0] / EXT[0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])
    u = 0.2 * np.stack([-0.05 * X[:, 0] + 0.02 * s, 0.03 * s, 0.01 * X[:, 0] ** 2], 1).ravel()
    u[P.op.mask != 0] = 0
    x = np.sin(0.37 * np.arange(P.op.size))
    P.op.apply_residual(u)
    y = P.op.apply_jacobian(x)
    return P, u, x, y


def _slice(field, npd_g, slab):
    nxg, nyg, nzg = npd_g
    v = field.reshape(nzg, nyg, nxg, 3)
    nx = slab.npd[0]
    return np.ascontiguousarray(v[:, :, slab.node_x0:slab.node_x0 + nx, :]).ravel()


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        Pg, u, x, yg = _global_fields()
        slab = slab_partition(GLOBAL_CELLS, world, rank, ORDER)
        h = EXT[0] / GLOBAL_CELLS[0]
        ext = (h * slab.cells[0], EXT[1], EXT[2])
        fixed = (0,) if rank == 0 else ()
        P = H.make_problem(ext, slab.cells, ORDER, fixed_faces=fixed)
        npd_g = Pg.mesh.npd
        ul, xl, yl_ref = _slice(u, npd_g, slab), _slice(x, npd_g, slab), _slice(yg, npd_g, slab)
        P.op.apply_residual(ul)
        y = torch.from_numpy(P.op.apply_jacobian(xl))
        exchange_faces(y, slab.npd, rank, world, dist)
        err = float(np.abs(y.numpy() - yl_ref).max() / np.abs(yl_ref).max())
        own = owned_mask(slab.npd, rank, world)
        d = global_dot(torch.from_numpy(xl), y, own, dist)
        # shared plane bitwise identical on both sides
        nx = slab.npd[0]
        v = y.view(slab.npd[2], slab.npd[1], nx, 3)
        plane = v[:, :, nx - 1, :].contiguous() if rank == 0 else v[:, :, 0, :].contiguous()
        other = torch.empty_like(plane)
        if rank == 0:
            dist.send(plane, 1)
            dist.recv(other, 1)
        else:
            dist.recv(other, 0)
            dist.send(plane, 0)
        out[rank] = (err, d, float(x @ yg), bool(torch.equal(plane, other)))
    finally:
        dist.destroy_process_group()


def test_slab_partition_shapes():
    s = [slab_partition((96, 48, 48), 8, r, 2) for r in range(8)]
    assert sum(x.cells[0] for x in s) == 96 and all(x.cells[0] == 12 for x in s)
    assert [x.x0 for x in s] == [12 * r for r in range(8)]
    s = [slab_partition((7, 3, 3), 3, r, 1) for r in range(3)]
    assert [x.cells[0] for x in s] == [3, 2, 2]
    with pytest.raises(ValueError):
        slab_partition((2, 2, 2), 3, 0, 2)


def test_two_rank_slab_apply_matches_global():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        err, d, dref, same = out[r]
        assert err < 1e-12
        assert abs(d - dref) < 1e-12 * abs(dref)
        assert same
