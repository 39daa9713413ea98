"""Slab-partitioned p-MG PCG (paper_2204_01722_b200.distributed) on CPU with
gloo, world sizes 1 and 2.  The level operations come from the numpy oracle
(checker only); the distributed composition under test is the product code:
interface exchange, interface-scaled transfers, global-seed lambda_max,
summed + replicated coarse factorisation, owned dots, natural-norm PCG.
It must reproduce the single-process reference algorithm (oracle Hierarchy
+ cg_solve) on the whole box: the same lambda_max per level (partition
independent by construction), the same PCG iteration count and solution."""
import os
import socket

import numpy as np
import pytest
import scipy.linalg as sla
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import hexmg_np as H
from dist_model import (DistributedHierarchy, SlabComm, distributed_pcg,
                                               distributed_solve, global_rough_seed_slice,
                                               q1_lattice_pattern)
from dist_partition_model import slab_partition

EXT = (3.0, 1.0, 1.0)
TRACTION = (0.0, 0.0, -0.02)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


class _DenseChol:
    def __init__(self, row_ptr, cols, npd):
        self.rp, self.cols = np.asarray(row_ptr), np.asarray(cols)
        self.n = len(self.rp) - 1

    def factorize(self, vals):
        A = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.rp))
        A[rows, self.cols] = vals
        self.c = sla.cho_factor(A, lower=True)

    def solve(self, b):
        return torch.from_numpy(sla.cho_solve(self.c, b.numpy()))


class OracleSlabBackend:
    """Level operations of one slab from the numpy oracle (test checker)."""

    def __init__(self, prob, fixed):
        self.prob = prob
        self.h = H.Hierarchy(prob.extents, prob.counts, prob.mesh.order, prob.basis.q, fixed,
                             prob.mu, prob.lam, prob.op)
        self.levels = [op.mesh.order for op in self.h.levels]
        self.device = torch.device("cpu")

    def size(self, k):
        return self.h.levels[k].size

    def npd(self, k):
        return tuple(self.h.levels[k].mesh.npd)

    def mask(self, k):
        return torch.from_numpy(self.h.levels[k].mask != 0)

    def apply(self, k, x):
        return torch.from_numpy(self.h.levels[k].apply_jacobian(x.numpy()))

    def diagonal(self, k):
        return torch.from_numpy(self.h.levels[k].extract_diagonal())

    def prolong(self, kc, xc):
        return torch.from_numpy(self.h.transfers[kc + 1].apply(xc.numpy()))

    def restrict(self, kc, xf):
        return torch.from_numpy(self.h.transfers[kc + 1].apply_transpose(xf.numpy()))

    def coarse_csr(self):
        op = self.h.levels[0]
        A = op.assemble_dense()
        rp, cols = q1_lattice_pattern(self.npd(0), op.mask)
        rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
        return rp, cols, A[rows, cols]

    def coarse_solver(self, row_ptr, cols, npd):
        return _DenseChol(row_ptr, cols, npd)

    def residual(self, u):
        return torch.from_numpy(self.prob.op.apply_residual(u.numpy()))

    def set_time(self, t):
        self.prob.op.load_scale = t


def _global_reference(cells, order):
    P = H.make_problem(EXT, cells, order, fixed_faces=(0,), traction_face=1, traction=TRACTION)
    f = P.op.apply_residual(np.zeros(P.op.size))
    hier = H.Hierarchy(EXT, cells, order, order + 1, (0,), P.mu, P.lam, P.op)
    hier.setup_numeric()
    b = -f
    rep = H.cg_solve(P.op.apply_jacobian, hier.precondition, b, np.zeros_like(b), 1e-10, 200)
    x = np.zeros_like(b)
    rep = H.cg_solve(P.op.apply_jacobian, hier.precondition, b, x, 1e-8, 200)
    lams = [s.lambda_max for s in hier.smoothers[1:]]
    return P, x, rep.iterations, lams


def _slice(field, npd_g, node_x0, nx):
    v = field.reshape(npd_g[2], npd_g[1], npd_g[0], 3)
    return np.ascontiguousarray(v[:, :, node_x0:node_x0 + nx, :]).ravel()


def _worker(rank, world, port, cells, order, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_default_dtype(torch.float64)
        slab = slab_partition(cells, world, rank, order)
        h = EXT[0] / cells[0]
        ext = (h * slab.cells[0], EXT[1], EXT[2])
        fixed = (0,) if rank == 0 else ()
        tface = 1 if rank == world - 1 else -1
        P = H.make_problem(ext, slab.cells, order, fixed_faces=fixed, traction_face=tface,
                           traction=TRACTION)
        comm = SlabComm(rank, world, dist)
        f = torch.from_numpy(P.op.apply_residual(np.zeros(P.op.size)))
        comm.exchange(f, slab.npd)
        b = -f
        be = OracleSlabBackend(P, fixed)

        def gmask(p):
            return H.build_constraints(H.build_box_mesh(EXT, cells, p), (0,))

        hier = DistributedHierarchy(be, comm, cells, slab.x0, gmask)
        hier.setup_numeric()
        rep = distributed_pcg(hier, b, rtol=1e-8)
        out[rank] = (rep["iterations"], rep["x"].numpy(), hier.lambda_max[1:], slab.node_x0,
                     slab.npd[0], rep["eig_max"] / rep["eig_min"])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_distributed_pmg_pcg_matches_single_process(world):
    cells, order = (6, 2, 2), 2
    Pg, xg, its_g, lams_g = _global_reference(cells, order)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), cells, order, out), nprocs=world, join=True)
    npd_g = Pg.mesh.npd
    for r in range(world):
        its, x, lams, x0, nx, cond = out[r]
        assert abs(its - its_g) <= 1, (its, its_g)
        for a, b in zip(lams, lams_g):
            assert abs(a - b) < 1e-10 * abs(b), (lams, lams_g)
        xr = _slice(xg, npd_g, x0, nx)
        assert np.linalg.norm(x - xr) < 1e-6 * np.linalg.norm(xr)


def test_three_rank_q3_hierarchy():
    """Three levels (Q3 -> Q2 -> Q1) over three slabs of unequal width."""
    cells, order, world = (7, 2, 2), 3, 3
    Pg, xg, its_g, lams_g = _global_reference(cells, order)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), cells, order, out), nprocs=world, join=True)
    for r in range(world):
        its, x, lams, x0, nx, cond = out[r]
        assert abs(its - its_g) <= 1
        assert len(lams) == len(lams_g) == 2
        for a, b in zip(lams, lams_g):
            assert abs(a - b) < 1e-10 * abs(b)
        xr = _slice(xg, Pg.mesh.npd, x0, nx)
        assert np.linalg.norm(x - xr) < 1e-6 * np.linalg.norm(xr)


def test_global_seed_slices_tile_the_global_seed():
    gnpd = (9, 3, 3)
    full = global_rough_seed_slice(gnpd, 0, gnpd)
    assert np.array_equal(full, H.rough_seed(3 * 81))
    a = global_rough_seed_slice(gnpd, 0, (5, 3, 3))
    b = global_rough_seed_slice(gnpd, 4, (5, 3, 3))
    g = full.reshape(3, 3, 9, 3)
    assert np.array_equal(a.reshape(3, 3, 5, 3), g[:, :, :5])
    assert np.array_equal(b.reshape(3, 3, 5, 3), g[:, :, 4:])


def test_q1_pattern_matches_assembled_operator():
    P = H.make_problem((1.0, 1.0, 1.0), (3, 2, 2), 1, fixed_faces=(0,))
    P.op.apply_residual(np.zeros(P.op.size))
    A = P.op.assemble_dense()
    rp, cols = q1_lattice_pattern(P.mesh.npd, P.op.mask)
    nz_rows, nz_cols = np.nonzero(A)
    pat = set(zip(np.repeat(np.arange(len(rp) - 1), np.diff(rp)).tolist(), cols.tolist()))
    assert set(zip(nz_rows.tolist(), nz_cols.tolist())) <= pat
    for i in range(len(rp) - 1):
        assert np.all(np.diff(cols[rp[i]:rp[i + 1]]) > 0)


def _newton_worker(rank, world, port, traction, steps, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_default_dtype(torch.float64)
        cells, order, ext = (4, 2, 2), 2, (2.0, 1.0, 1.0)
        slab = slab_partition(cells, world, rank, order)
        h = ext[0] / cells[0]
        fixed = (0,) if rank == 0 else ()
        P = H.make_problem((h * slab.cells[0], ext[1], ext[2]), slab.cells, order,
                           fixed_faces=fixed, traction_face=1 if rank == world - 1 else -1,
                           traction=traction)
        hier = DistributedHierarchy(OracleSlabBackend(P, fixed), SlabComm(rank, world, dist),
                                    cells, slab.x0,
                                    lambda p: H.build_constraints(H.build_box_mesh(ext, cells, p), (0,)))
        rep = distributed_solve(hier, load_steps=steps, use_line_search=False)
        out[rank] = (rep["newton_iterations"], rep["cg_iterations"], rep["final_fnorm"],
                     rep["u"].numpy(), slab.node_x0, slab.npd[0])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case,traction,steps", [("compress1_ls0", (-0.05, 0.0, 0.0), 1),
                                                 ("bend_ls0", (0.0, 0.0, -0.02), 5)])
def test_distributed_newton_matches_reference(case, traction, steps):
    """Slab-partitioned Newton + p-MG + load continuation (2 ranks) against
    the UNMODIFIED reference's FemProblem::solve on the whole bar
    (tests/golden/newton.npz): iteration counts and the solution."""
    G = np.load(os.path.join(os.path.dirname(__file__), "golden", "newton.npz"))
    ni, ci, fn = G[f"{case}_stats"]
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_newton_worker, args=(2, _free_port(), traction, steps, out), nprocs=2, join=True)
    npd_g = (9, 5, 5)
    for r in range(2):
        its, cgits, fnorm, u, x0, nx = out[r]
        assert abs(its - ni) <= steps and abs(cgits - ci) <= its
        assert fnorm < 1e-9
        ur = _slice(G[f"{case}_u"], npd_g, x0, nx)
        assert np.linalg.norm(u - ur) < 1e-9 * np.linalg.norm(ur)


def _block_worker(rank, world, port, cells, order, dims, out):
    from dist_model import BlockComm
    from dist_partition_model import block_partition
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_default_dtype(torch.float64)
        blk = block_partition(cells, dims, rank, order)
        h = [EXT[d] / cells[d] for d in range(3)]
        ext = tuple(h[d] * blk.cells[d] for d in range(3))
        fixed = (0,) if blk.coords[0] == 0 else ()
        tface = 1 if blk.coords[0] == dims[0] - 1 else -1
        P = H.make_problem(ext, blk.cells, order, fixed_faces=fixed, traction_face=tface,
                           traction=TRACTION)
        comm = BlockComm(blk, dist)
        f = torch.from_numpy(P.op.apply_residual(np.zeros(P.op.size)))
        comm.exchange(f, blk.npd)
        be = OracleSlabBackend(P, fixed)

        def gmask(p):
            return H.build_constraints(H.build_box_mesh(EXT, cells, p), (0,))

        hier = DistributedHierarchy(be, comm, cells, blk.e0, gmask)
        hier.setup_numeric()
        rep = distributed_pcg(hier, -f, rtol=1e-8)
        out[rank] = (rep["iterations"], rep["x"].numpy(), hier.lambda_max[1:], blk.node0, blk.npd)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(2, 2, 1), (1, 2, 2)])
def test_block_partitioned_pmg_matches_single_process(dims):
    """px x py x pz block partition (SURVEY.md §8(e), 2 x 2 x 2 for cfg5):
    interface sums through edges and corners, per-direction interface
    scaling of the transfers, ownership by the lower block; same lambda_max,
    PCG iterations and solution as the single-process reference."""
    cells, order = (6, 4, 4), 2
    world = dims[0] * dims[1] * dims[2]
    Pg, xg, its_g, lams_g = _global_reference(cells, order)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_block_worker, args=(world, _free_port(), cells, order, dims, out), nprocs=world,
             join=True)
    g = xg.reshape(Pg.mesh.npd[2], Pg.mesh.npd[1], Pg.mesh.npd[0], 3)
    for r in range(world):
        its, x, lams, n0, npd = out[r]
        assert abs(its - its_g) <= 1, (its, its_g)
        for a, b in zip(lams, lams_g):
            assert abs(a - b) < 1e-10 * abs(b), (lams, lams_g)
        xr = np.ascontiguousarray(g[n0[2]:n0[2] + npd[2], n0[1]:n0[1] + npd[1],
                                    n0[0]:n0[0] + npd[0]]).ravel()
        assert np.linalg.norm(x - xr) < 1e-6 * np.linalg.norm(xr)


def test_block_partition_shapes():
    from dist_partition_model import block_partition
    bs = [block_partition((160, 160, 160), (2, 2, 2), r, 2) for r in range(8)]
    assert all(b.cells == (80, 80, 80) for b in bs)
    assert sorted(b.e0 for b in bs) == sorted((x, y, z) for x in (0, 80) for y in (0, 80)
                                              for z in (0, 80))
    b = block_partition((7, 5, 3), (3, 2, 1), 4, 1)
    assert b.coords == (1, 1, 0) and b.cells == (2, 2, 3) and b.e0 == (3, 3, 0)
    assert b.neighbour(0, -1) == 3 and b.neighbour(0, 1) == 5 and b.neighbour(1, 1) is None
