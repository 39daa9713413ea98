"""Partitioned (multi-GPU) p-multigrid through the C-ABI.

The reference is single-process; the paper distributes the same
operator, summing shared nodes after every apply (A = P^T E^T B^T D B E P,
PAPER.md:224-228, :316).  The whole composition -- interface sums, owned
dots, interface-scaled transfers, global-seed lambda_max, the coarse level,
PCG and Newton -- lives in the C++ library (csrc/dist.cu, csrc/solver.cpp,
``hxg_mg_create_partitioned``).  This module only launches it:

* ``Communicator``: the library's built-in NCCL communicator (unique id from
  rank 0, broadcast over the caller's process group) or a table of ctypes
  callbacks over a torch.distributed process group (gloo: the host-staged
  path the multi-process tests on one GPU use);
* ``PartitionedProblem``: this rank's block of the box (``hxg_partition_block``),
  its FemProblem (geometry, Dirichlet faces and traction on the block) and the
  partitioned hierarchy, with the solver entry points.
"""
from __future__ import annotations

import ctypes
import traceback

import numpy as np
import torch

from . import capi
from .capi import check, lib
from .hexmg import FemProblem, _dev, _out, _ptr, _report, newton_config

FACES = {"-x": 0, "+x": 1, "-y": 2, "+y": 3, "-z": 4, "+z": 5}

_EXCH = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                         ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_void_p),
                         ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p)
_ALLRED = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                           ctypes.c_int, ctypes.c_void_p)


class _CommOps(ctypes.Structure):
    _fields_ = [("ctx", ctypes.c_void_p), ("exchange", _EXCH), ("allreduce", _ALLRED)]


def partition_block(global_cells, dims, rank):
    """This rank's block: (local element counts, first global element)."""
    g = (ctypes.c_int * 3)(*global_cells)
    d = (ctypes.c_int * 3)(*dims)
    cells, e0 = (ctypes.c_int * 3)(), (ctypes.c_int * 3)()
    check(lib().hxg_partition_block(g, d, int(rank), cells, e0))
    return tuple(cells), tuple(e0)


class Communicator:
    """hxg_comm_t: NCCL (built in) or callbacks over a torch process group."""

    def __init__(self, rank, world, dist=None, backend="nccl"):
        self.rank, self.world, self.dist = rank, world, dist
        h = ctypes.c_void_p()
        if backend == "nccl":
            uid = (ctypes.c_ubyte * 128)()
            if rank == 0:
                check(lib().hxg_nccl_unique_id(ctypes.cast(uid, ctypes.c_void_p)))
            if world > 1:
                t = torch.tensor(list(uid), dtype=torch.uint8,
                                 device="cuda" if dist.get_backend() == "nccl" else "cpu")
                dist.broadcast(t, 0)
                uid = (ctypes.c_ubyte * 128)(*t.cpu().tolist())
            check(lib().hxg_comm_create_nccl(rank, world, ctypes.cast(uid, ctypes.c_void_p), ctypes.byref(h)))
        else:
            self._ops = _CommOps(None, _EXCH(self._exchange), _ALLRED(self._allreduce))
            check(lib().hxg_comm_create(rank, world, ctypes.byref(self._ops), ctypes.byref(h)))
        self.h = h

    # host-staged collectives over the process group (gloo)
    def _d2h(self, ptr, n):
        a = np.empty(n, np.float64)
        check(lib().hxg_memcpy_d2h(a.ctypes.data, ptr, n * 8))
        return torch.from_numpy(a)

    def _h2d(self, ptr, t):
        a = np.ascontiguousarray(t.numpy())
        check(lib().hxg_memcpy_h2d(ptr, a.ctypes.data, a.size * 8))

    def _exchange(self, ctx, npeers, peers, send, recv, counts, stream):
        try:
            check(lib().hxg_stream_synchronize(stream))
            ops, bufs = [], []
            for i in range(npeers):
                n = int(counts[i])
                s = self._d2h(send[i], n)
                r = torch.empty(n, dtype=torch.float64)
                ops += [self.dist.P2POp(self.dist.isend, s, int(peers[i])),
                        self.dist.P2POp(self.dist.irecv, r, int(peers[i]))]
                bufs.append((r, recv[i]))
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
            for r, dst in bufs:
                self._h2d(dst, r)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed call
            traceback.print_exc()
            return 1

    def _allreduce(self, ctx, data, count, op, stream):
        try:
            check(lib().hxg_stream_synchronize(stream))
            t = self._d2h(data, int(count))
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op else self.dist.ReduceOp.SUM)
            self._h2d(data, t)
            return 0
        except Exception:  # noqa: BLE001
            traceback.print_exc()
            return 1

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().hxg_comm_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None


class PartitionedProblem:
    """This rank's block of a FemProblem on the box of ``global_cells``
    elements cut into ``dims`` blocks, with the partitioned p-MG hierarchy.
    Vectors are this block's local L-vectors (shared interface entries equal
    on every rank holding them)."""

    def __init__(self, comm: Communicator, global_cells, dims, order=2, extents=(1.0, 1.0, 1.0),
                 fixed_faces=("-x",), traction_face=None, traction=(0.0, 0.0, 0.0),
                 geometry="box", **fem):
        self.comm, self.global_cells, self.dims = comm, tuple(global_cells), tuple(dims)
        self.cells, self.e0 = partition_block(global_cells, dims, comm.rank)
        coords = (comm.rank % dims[0], (comm.rank // dims[0]) % dims[1],
                  comm.rank // (dims[0] * dims[1]))
        on = lambda f: coords[FACES[f] // 2] == (0 if FACES[f] % 2 == 0 else dims[FACES[f] // 2] - 1)  # noqa: E731
        local_ext = tuple(extents[d] * self.cells[d] / global_cells[d] for d in range(3))
        self.prob = FemProblem(extents=local_ext, cells=self.cells, order=order,
                               fixed_faces=tuple(f for f in fixed_faces if on(f)),
                               traction_face=traction_face if traction_face and on(traction_face)
                               else None, traction=traction, geometry=geometry, **fem)
        self.op = self.prob.op
        self.global_faces = sum(1 << FACES[f] for f in fixed_faces)
        h = ctypes.c_void_p()
        check(lib().hxg_mg_create_partitioned(self.op.h, comm.h, (ctypes.c_int * 3)(*global_cells),
                                              (ctypes.c_int * 3)(*dims), self.global_faces, None,
                                              0, 1, 1, ctypes.byref(h)))
        self.h = h
        n = ctypes.c_int()
        check(lib().hxg_mg_num_levels(self.h, ctypes.byref(n)))
        self.levels = n.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().hxg_mg_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def size(self, level=None):
        n = ctypes.c_int64()
        check(lib().hxg_mg_level_size(self.h, self.levels - 1 if level is None else level,
                                      ctypes.byref(n)))
        return n.value

    def apply(self, x, y=None, level=None):
        k = self.levels - 1 if level is None else level
        n = self.size(k)
        x = _dev(x, n)
        y = torch.empty_like(x) if y is None else _out(y, n)
        check(lib().hxg_mg_apply(self.h, k, _ptr(x), _ptr(y)))
        return y

    def residual(self, u, f=None):
        n = self.size()
        u = _dev(u, n)
        f = torch.empty_like(u) if f is None else _out(f, n)
        check(lib().hxg_mg_residual(self.h, _ptr(u), _ptr(f)))
        return f

    def dot(self, x, y, level=None):
        k = self.levels - 1 if level is None else level
        out = ctypes.c_double()
        check(lib().hxg_mg_dot(self.h, k, _ptr(_dev(x, self.size(k))), _ptr(_dev(y, self.size(k))),
                               ctypes.byref(out)))
        return out.value

    def setup_numeric(self):
        check(lib().hxg_mg_setup_numeric(self.h))

    def set_coarse_mode(self, mode):
        m = {"auto": 0, "dense": 1, "nd": 2, "hmg": 4}.get(mode, mode)
        check(lib().hxg_mg_set_coarse_mode(self.h, int(m)))

    def lambda_max(self, k):
        out = ctypes.c_double()
        check(lib().hxg_mg_lambda_max(self.h, k, ctypes.byref(out)))
        return out.value

    def v_cycle(self, b, x=None):
        b = _dev(b, self.size())
        x = torch.zeros_like(b) if x is None else _out(x, self.size())
        check(lib().hxg_mg_vcycle(self.h, _ptr(b), _ptr(x)))
        return x

    def cg_solve(self, b, x=None, rtol=1e-8, max_iterations=500, precond="mg"):
        pc = {"none": 0, "jacobi": 1, "mg": 2}[precond]
        b = _dev(b, self.size())
        x = torch.zeros_like(b) if x is None else _out(x, self.size())
        rep = capi.CgReport()
        hist = np.zeros(max_iterations + 2)
        check(lib().hxg_cg_solve(self.op.h, self.h, pc, _ptr(b), _ptr(x), rtol, max_iterations,
                                 ctypes.byref(rep), _ptr(hist), len(hist)))
        return dict(x=x, iterations=rep.iterations, converged=bool(rep.converged),
                    eig_min=rep.eig_min, eig_max=rep.eig_max,
                    history=hist[: rep.iterations + 1].copy())

    def solve(self, max_bisections=3, **config):
        """FemProblem::solve (problem.hpp:118-127) on the partitioned system."""
        u = torch.zeros(self.size(), dtype=torch.float64, device="cuda")
        cfg = newton_config(**config)
        rep = capi.SolveReport()
        recs = (capi.IterationRecord * 2048)()
        check(lib().hxg_solve_continuation(self.op.h, self.h, ctypes.byref(cfg), _ptr(u),
                                           int(max_bisections), ctypes.byref(rep), recs, 2048))
        out = _report(rep, recs)
        out["u"] = u
        return out
