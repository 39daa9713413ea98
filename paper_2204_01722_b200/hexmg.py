"""Python mirror of the reference ``hexmg`` operator API over the C-ABI.

Names, argument meaning and error behaviour follow the reference headers
(/root/reference/proj/include/hexmg): ``MatrixFreeOperator`` (operator.hpp:70),
``MultigridHierarchy`` / ``build_hierarchy`` (multigrid.hpp:88, :212),
``cg_solve`` (cg.hpp:81), ``FemProblem`` (problem.hpp:19).  Vectors are CUDA
``torch.float64`` tensors (torch is only the device-memory plumbing); every
operation is a call into libhexmg_b200.so.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import capi
from .capi import check, lib

FACES = {"-x": 0, "+x": 1, "-y": 2, "+y": 3, "-z": 4, "+z": 5}


def _ptr(a) -> ctypes.c_void_p:
    if isinstance(a, torch.Tensor):
        return ctypes.c_void_p(a.data_ptr())
    if isinstance(a, np.ndarray):
        return a.ctypes.data_as(ctypes.c_void_p)
    if a is None:
        return ctypes.c_void_p(None)
    raise TypeError(type(a))


def _dev(t, n=None) -> torch.Tensor:
    t = torch.as_tensor(t, dtype=torch.float64)
    if not t.is_cuda:
        t = t.cuda()
    t = t.contiguous()
    if n is not None and t.numel() != n:
        raise ValueError("nodal field size mismatch")
    return t


def _out(t, n) -> torch.Tensor:
    """Caller-supplied output buffer: the device kernels write n float64
    entries through its pointer, so anything else is refused up front."""
    if not isinstance(t, torch.Tensor):
        raise ValueError("output buffer must be a torch tensor")
    if t.dtype != torch.float64 or not t.is_cuda or not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"output buffer must be a contiguous float64 CUDA tensor of {n} entries "
                         f"(got {t.dtype}, {t.device}, contiguous={t.is_contiguous()}, "
                         f"numel={t.numel()})")
    return t


@dataclass
class Basis1D:
    """basis.hpp:117-130 (host tabulations from the library's setup)."""

    order: int
    q: int
    nodes: np.ndarray
    points: np.ndarray
    weights: np.ndarray
    interp: np.ndarray
    deriv: np.ndarray
    pinv: np.ndarray
    colloc: np.ndarray


def build_lagrange_basis(p: int, q: int | None = None) -> Basis1D:
    q = q or p + 1
    n = p + 1
    arr = dict(nodes=np.zeros(n), points=np.zeros(q), weights=np.zeros(q), interp=np.zeros((q, n)),
               deriv=np.zeros((q, n)), pinv=np.zeros((n, q)), colloc=np.zeros((q, q)))
    check(lib().hxg_setup_basis(p, q, *[_ptr(arr[k]) for k in
                                        ("nodes", "points", "weights", "interp", "deriv", "pinv",
                                         "colloc")]))
    return Basis1D(p, q, **arr)


def lame_from_young_poisson(young: float, poisson: float):
    """material.hpp:27-36."""
    if not young > 0.0:
        raise ValueError("Young's modulus must be positive")
    if poisson == 0.5:
        raise ValueError("incompressible limit nu = 0.5 is unsupported")
    if not (-1.0 < poisson < 0.5):
        raise ValueError("Poisson ratio must lie in (-1, 0.5)")
    mu = young / (2.0 * (1.0 + poisson))
    lam = young * poisson / ((1.0 + poisson) * (1.0 - 2.0 * poisson))
    return mu, lam


def num_nodes(cells, order):
    return (order * cells[0] + 1) * (order * cells[1] + 1) * (order * cells[2] + 1)


def geometric_factors(extents, cells, order, q):
    """compute_geometric_factors (mesh.hpp:193-232): (E, q^3, 3, 3), (E, q^3)."""
    E = cells[0] * cells[1] * cells[2]
    dx = np.zeros((E, q**3, 3, 3))
    w = np.zeros((E, q**3))
    check(lib().hxg_setup_geometry(_ptr(np.asarray(extents, np.float64)),
                                   _ptr(np.asarray(cells, np.int32)), order, q, _ptr(dx), _ptr(w)))
    return dx, w


def constraint_mask(cells, order, fixed_faces):
    """build_constraints (operator.hpp:36-55) for whole-face Dirichlet sets."""
    m = np.zeros(3 * num_nodes(cells, order), dtype=np.uint8)
    fm = 0
    for f in fixed_faces:
        fm |= 1 << FACES[f]
    check(lib().hxg_setup_constraints(_ptr(np.asarray(cells, np.int32)), order, fm, _ptr(m)))
    return m, fm


def traction_load(extents, cells, order, q, face, traction):
    """assemble_traction_load (operator.hpp:381-443)."""
    load = np.zeros(3 * num_nodes(cells, order))
    if face is None:
        return load
    check(lib().hxg_setup_traction_load(_ptr(np.asarray(extents, np.float64)),
                                        _ptr(np.asarray(cells, np.int32)), order, q, FACES[face],
                                        _ptr(np.asarray(traction, np.float64)), _ptr(load)))
    return load


# JacobianStorage (material.hpp:66-78) by its config name (config.hpp:193-198)
# and the reference's per-point state scalars.
STORAGES = {"current": 0, "initial-native": 1, "initial-tuned": 2, "initial-ad": 3}
STATE_SCALARS = {0: 17, 1: 19, 2: 26, 3: 25}


def storage_id(storage):
    if isinstance(storage, str):
        if storage not in STORAGES:
            raise ValueError(f"unknown jacobian storage '{storage}'")
        return STORAGES[storage]
    return int(storage)


def body_force_load(extents, cells, basis: Basis1D, force):
    """assemble_body_force_load (operator.hpp:440-456) for the box mesh:
    load[node, c] = f_c sum_e sum_q w detJ N_a(q).  The box map is affine and
    tensor-product, so the assembled vector is f_c detJ (m_x x m_y x m_z) with
    m_d the assembled 1D vectors sum_i w_i B[i, a] (host setup, once)."""
    p, q = basis.order, basis.q
    B = np.asarray(basis.interp).reshape(q, p + 1)
    s = np.asarray(basis.weights) @ B  # (p+1,) 1D element integrals
    ms = []
    for d in range(3):
        m = np.zeros(p * cells[d] + 1)
        for e in range(cells[d]):
            m[p * e:p * e + p + 1] += s
        ms.append(m)
    detj = np.prod([extents[d] / (2.0 * cells[d]) for d in range(3)])
    nodal = detj * np.einsum("k,j,i->kji", ms[2], ms[1], ms[0]).ravel()
    return np.ascontiguousarray((nodal[:, None] * np.asarray(force, np.float64)[None, :]).ravel())


class MatrixFreeOperator:
    """MatrixFreeOperator (operator.hpp:70-373) on the GPU."""

    def __init__(self, cells, basis: Basis1D, dxidX, weight, mu, lam, mask=None, state=None,
                 _handle=None, extents=None, storage=0):
        self._owner = _handle is None
        self.storage = storage_id(storage)
        if _handle is not None:
            self.h = _handle
        else:
            self._keep = [np.ascontiguousarray(basis.interp), np.ascontiguousarray(basis.deriv),
                          np.ascontiguousarray(basis.colloc)]
            desc = capi.OpDesc()
            desc.order, desc.qpts = basis.order, basis.q
            desc.cells[:] = list(cells)
            desc.interp, desc.deriv, desc.colloc = [_ptr(a).value for a in self._keep]
            if dxidX is not None:
                dx = np.ascontiguousarray(dxidX, np.float64)
                w = np.ascontiguousarray(weight, np.float64)
                self._keep += [dx, w]
                desc.dxidX, desc.weight = _ptr(dx).value, _ptr(w).value
            elif extents is not None:  # affine box geometry computed on the device
                ext = np.ascontiguousarray(extents, np.float64)
                qw = np.ascontiguousarray(basis.weights, np.float64)
                self._keep += [ext, qw]
                desc.extents, desc.qweights = _ptr(ext).value, _ptr(qw).value
            desc.mu, desc.lam, desc.storage = mu, lam, self.storage
            if mask is not None:
                m = np.ascontiguousarray(mask, np.uint8)
                self._keep.append(m)
                desc.mask = _ptr(m).value
            h = ctypes.c_void_p()
            check(lib().hxg_op_create(ctypes.byref(desc), state, ctypes.byref(h)))
            self.h = h
        n = ctypes.c_int64()
        check(lib().hxg_op_size(self.h, ctypes.byref(n)))
        self._size = n.value

    def __del__(self):
        if getattr(self, "_owner", False) and getattr(self, "h", None):
            try:
                lib().hxg_op_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def size(self) -> int:
        return self._size

    def set_external_load(self, load):
        load = np.ascontiguousarray(load, np.float64) if load is not None else None
        check(lib().hxg_op_set_external_load(self.h, _ptr(load)))

    def set_load_scale(self, s):
        check(lib().hxg_op_set_load_scale(self.h, float(s)))

    def set_jacobian_perturbation(self, eps):
        check(lib().hxg_op_set_jacobian_perturbation(self.h, float(eps)))

    def set_variant(self, v: int):
        check(lib().hxg_op_set_variant(self.h, int(v)))

    def kernel_launches(self) -> int:
        n = ctypes.c_int()
        check(lib().hxg_op_kernel_launches(self.h, ctypes.byref(n)))
        return n.value

    def stored_bytes_per_dof(self) -> float:
        out = ctypes.c_double()
        check(lib().hxg_op_stored_bytes_per_dof(self.h, ctypes.byref(out)))
        return out.value

    def counters(self):
        r, j = ctypes.c_int64(), ctypes.c_int64()
        check(lib().hxg_op_counters(self.h, ctypes.byref(r), ctypes.byref(j)))
        return r.value, j.value

    def apply_residual(self, u, out=None):
        u = _dev(u, self._size)
        out = torch.empty_like(u) if out is None else _out(out, self._size)
        check(lib().hxg_op_apply_residual(self.h, _ptr(u), _ptr(out)))
        return out

    def apply_jacobian(self, du, out=None):
        du = _dev(du, self._size)
        out = torch.empty_like(du) if out is None else _out(out, self._size)
        check(lib().hxg_op_apply_jacobian(self.h, _ptr(du), _ptr(out)))
        return out

    def apply_jacobian_host(self, du: np.ndarray, out: np.ndarray | None = None):
        du = np.ascontiguousarray(du, np.float64)
        if du.size != self._size:
            raise ValueError("nodal field size mismatch")
        if out is None:
            out = np.empty_like(du)
        elif not (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.size == self._size
                  and out.flags.c_contiguous and out.flags.writeable):
            raise ValueError("host output must be a writeable contiguous float64 array of op.size()")
        check(lib().hxg_op_apply_jacobian_host(self.h, _ptr(du), _ptr(out)))
        return out

    def extract_diagonal(self, out=None):
        out = (torch.empty(self._size, dtype=torch.float64, device="cuda") if out is None
               else _out(out, self._size))
        check(lib().hxg_op_extract_diagonal(self.h, _ptr(out)))
        return out

    def total_strain_energy(self, u) -> float:
        u = _dev(u, self._size)
        e = ctypes.c_double()
        check(lib().hxg_op_total_strain_energy(self.h, _ptr(u), ctypes.byref(e)))
        return e.value

    def export_state(self, num_elements, nq):
        out = np.zeros((num_elements, nq, STATE_SCALARS[self.storage]))
        check(lib().hxg_op_export_state(self.h, _ptr(out)))
        return out

    def gather(self, u, num_elements, npe):
        u = _dev(u, self._size)
        ev = torch.empty(num_elements * 3 * npe, dtype=torch.float64, device="cuda")
        check(lib().hxg_op_gather(self.h, _ptr(u), _ptr(ev)))
        return ev

    def scatter_add(self, ev, out):
        check(lib().hxg_op_scatter_add(self.h, _ptr(_dev(ev)), _ptr(_out(out, self._size))))
        return out

    def time_jacobian_parts(self, x, y, warmup=3, repeats=20):
        """(brick kernel ms, fix-up kernel ms) per fused apply, events on the stream."""
        ms = np.zeros(2)
        check(lib().hxg_op_time_jacobian_parts(self.h, _ptr(_dev(x, self.size())),
                                               _ptr(_out(y, self.size())), warmup, repeats, _ptr(ms)))
        return float(ms[0]), float(ms[1])

    def time_jacobian(self, x, y, warmup=3, repeats=20) -> float:
        ms = ctypes.c_double()
        x, y = _dev(x, self._size), _out(y, self._size)
        check(lib().hxg_op_time_jacobian(self.h, _ptr(x), _ptr(y), warmup, repeats, ctypes.byref(ms)))
        return ms.value


class MultigridHierarchy:
    """MultigridHierarchy + build_hierarchy (multigrid.hpp:88-268)."""

    def __init__(self, fine: MatrixFreeOperator, fixed_face_mask: int, schedule=None,
                 pre_smooth=1, post_smooth=1):
        self.fine = fine
        h = ctypes.c_void_p()
        sched = None if schedule is None else np.asarray(schedule, np.int32)
        check(lib().hxg_mg_create(fine.h, fixed_face_mask, _ptr(sched),
                                  0 if sched is None else len(sched), pre_smooth, post_smooth,
                                  ctypes.byref(h)))
        self.h = h
        n = ctypes.c_int()
        check(lib().hxg_mg_num_levels(self.h, ctypes.byref(n)))
        self._levels = n.value

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().hxg_mg_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def num_levels(self):
        return self._levels

    def level_size(self, k):
        n = ctypes.c_int64()
        check(lib().hxg_mg_level_size(self.h, k, ctypes.byref(n)))
        return n.value

    def level_operator(self, k) -> MatrixFreeOperator:
        h = ctypes.c_void_p()
        check(lib().hxg_mg_level_op(self.h, k, ctypes.byref(h)))
        op = MatrixFreeOperator(None, None, None, None, 0, 0, _handle=h, storage=self.fine.storage)
        op._hier = self  # keep the hierarchy alive
        return op

    def setup_numeric(self):
        check(lib().hxg_mg_setup_numeric(self.h))

    def assemble_coarse(self):
        """coo_numeric only (no smoothers / factorization)."""
        check(lib().hxg_mg_assemble_coarse(self.h))

    def set_coarse_mode(self, mode):
        """0 automatic, 1 dense (one front), 2 nested-dissection multifrontal,
        4 ("hmg") inexact: one Galerkin h-multigrid V-cycle on the p = 1 level."""
        mode = {"auto": 0, "dense": 1, "sparse": 2, "nd": 2, "hmg": 4}.get(mode, mode)
        check(lib().hxg_mg_set_coarse_mode(self.h, int(mode)))

    def lambda_max(self, k):
        out = ctypes.c_double()
        check(lib().hxg_mg_lambda_max(self.h, k, ctypes.byref(out)))
        return out.value

    def prolong(self, coarse_level, xc):
        xc = _dev(xc, self.level_size(coarse_level))
        xf = torch.empty(self.level_size(coarse_level + 1), dtype=torch.float64, device="cuda")
        check(lib().hxg_mg_prolong(self.h, coarse_level, _ptr(xc), _ptr(xf)))
        return xf

    def restrict_to(self, coarse_level, xf):
        xf = _dev(xf, self.level_size(coarse_level + 1))
        xc = torch.empty(self.level_size(coarse_level), dtype=torch.float64, device="cuda")
        check(lib().hxg_mg_restrict(self.h, coarse_level, _ptr(xf), _ptr(xc)))
        return xc

    def v_cycle(self, b, x=None):
        b = _dev(b, self.level_size(self.num_levels() - 1))
        x = torch.zeros_like(b) if x is None else _out(x, b.numel())
        check(lib().hxg_mg_vcycle(self.h, _ptr(b), _ptr(x)))
        return x

    def smooth(self, k, b, x):
        n = self.level_size(k)
        check(lib().hxg_mg_smooth(self.h, k, _ptr(_dev(b, n)), _ptr(_out(x, n))))
        return x

    def coarse_csr(self):
        nnz = ctypes.c_int64()
        check(lib().hxg_mg_coarse_nnz(self.h, ctypes.byref(nnz)))
        n = self.level_size(0)
        rp = np.zeros(n + 1, np.int32)
        cols = np.zeros(nnz.value, np.int32)
        vals = np.zeros(nnz.value)
        check(lib().hxg_mg_coarse_csr_host(self.h, _ptr(rp), _ptr(cols), _ptr(vals)))
        return rp, cols, vals

    def hmg_levels(self):
        """Number of h-multigrid levels of the inexact coarse mode (0 if inactive)."""
        k = ctypes.c_int()
        check(lib().hxg_mg_hmg_levels(self.h, ctypes.byref(k)))
        return k.value

    def hmg_level_csr(self, level):
        """(row_ptr, cols, vals, mask) of h-multigrid level `level`'s Galerkin matrix."""
        n, nnz = ctypes.c_int64(), ctypes.c_int64()
        check(lib().hxg_mg_hmg_level_nnz(self.h, int(level), ctypes.byref(n), ctypes.byref(nnz)))
        rp = np.zeros(n.value + 1, np.int32)
        cols = np.zeros(nnz.value, np.int32)
        vals = np.zeros(nnz.value)
        mask = np.zeros(n.value, np.uint8)
        check(lib().hxg_mg_hmg_level_csr_host(self.h, int(level), _ptr(rp), _ptr(cols), _ptr(vals),
                                              _ptr(mask)))
        return rp, cols, vals, mask

    def coarse_vals_device(self):
        """The assembled coarse values as a CUDA tensor (CSR order of coarse_csr)."""
        nnz = ctypes.c_int64()
        check(lib().hxg_mg_coarse_nnz(self.h, ctypes.byref(nnz)))
        v = torch.empty(nnz.value, dtype=torch.float64, device="cuda")
        check(lib().hxg_mg_coarse_vals_device(self.h, _ptr(v)))
        return v

    def coarse_solve(self, b):
        b = _dev(b, self.level_size(0))
        x = torch.empty_like(b)
        check(lib().hxg_mg_coarse_solve(self.h, _ptr(b), _ptr(x)))
        return x


class AssembledOperator:
    """CooAssembly (assembly.hpp:134-230) of a MatrixFreeOperator of any
    order on the device: CSR symbolic at construction, numeric() from the
    operator's current state, matvec = CsrMatrix::matvec."""

    def __init__(self, op: MatrixFreeOperator):
        self.op = op
        h = ctypes.c_void_p()
        check(lib().hxg_asm_create(op.h, ctypes.byref(h)))
        self.h = h
        nnz = ctypes.c_int64()
        check(lib().hxg_asm_nnz(self.h, ctypes.byref(nnz)))
        self.nnz = nnz.value
        self.n = op.size()

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().hxg_asm_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def numeric(self):
        check(lib().hxg_asm_numeric(self.h))

    def matvec(self, x, y=None):
        x = _dev(x, self.n)
        y = torch.empty_like(x) if y is None else _out(y, self.n)
        check(lib().hxg_asm_matvec(self.h, _ptr(x), _ptr(y)))
        return y

    def csr(self):
        rp = np.zeros(self.n + 1, np.int32)
        cols = np.zeros(self.nnz, np.int32)
        vals = np.zeros(self.nnz, np.float64)
        check(lib().hxg_asm_csr_host(self.h, _ptr(rp), _ptr(cols), _ptr(vals)))
        return rp, cols, vals


class CoarseCholesky:
    """CholeskyCoarseSolver (coarse_solver.hpp:16-47) on a caller-assembled
    Q1 lattice matrix: analyzePattern at construction, factorize(vals),
    solve(b) on device vectors."""

    def __init__(self, row_ptr, cols, npd, mode="auto"):
        mode = {"auto": 0, "dense": 1, "sparse": 2, "nd": 2}.get(mode, mode)
        self._rp = np.ascontiguousarray(row_ptr, np.int32)
        self._cols = np.ascontiguousarray(cols, np.int32)
        self.n = len(self._rp) - 1
        h = ctypes.c_void_p()
        check(lib().hxg_chol_create(self.n, _ptr(self._rp), _ptr(self._cols),
                                    _ptr(np.asarray(npd, np.int32)), int(mode), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            try:
                lib().hxg_chol_destroy(self.h)
            except Exception:  # interpreter shutdown
                pass
            self.h = None

    def factorize(self, vals):
        if isinstance(vals, torch.Tensor) and vals.is_cuda:
            if vals.numel() != self._cols.size:
                raise ValueError("value array does not match the pattern")
            check(lib().hxg_chol_factorize_device(self.h, _ptr(vals.contiguous())))
            return
        vals = np.ascontiguousarray(vals, np.float64)
        if vals.size != self._cols.size:
            raise ValueError("value array does not match the pattern")
        check(lib().hxg_chol_factorize(self.h, _ptr(vals)))

    def solve(self, b, x=None):
        b = _dev(b, self.n)
        x = torch.empty_like(b) if x is None else _out(x, self.n)
        check(lib().hxg_chol_solve(self.h, _ptr(b), _ptr(x)))
        return x


def cg_solve(op: MatrixFreeOperator, b, x=None, rtol=1e-8, max_iterations=500,
             precond="mg", mg: MultigridHierarchy | None = None):
    """cg_solve (cg.hpp:81-134); precond in {"none", "jacobi", "mg"}."""
    pc = {"none": 0, "jacobi": 1, "mg": 2}[precond]
    b = _dev(b, op.size())
    x = torch.zeros_like(b) if x is None else _out(x, op.size())
    rep = capi.CgReport()
    hist = np.zeros(max_iterations + 2)
    check(lib().hxg_cg_solve(op.h, mg.h if mg is not None else None, pc, _ptr(b), _ptr(x), rtol,
                             max_iterations, ctypes.byref(rep), _ptr(hist), len(hist)))
    return dict(x=x, iterations=rep.iterations, converged=bool(rep.converged),
                eig_min=rep.eig_min, eig_max=rep.eig_max,
                history=hist[: rep.iterations + 1].copy())


def newton_config(**overrides) -> capi.NewtonConfig:
    """NewtonConfig with the reference defaults (config.hpp:55-61) and
    keyword overrides (max_iterations, rtol, atol, linear_rtol,
    linear_max_iterations, use_line_search, load_steps,
    reference_line_search_quirk)."""
    cfg = capi.NewtonConfig()
    check(lib().hxg_newton_config_default(ctypes.byref(cfg)))
    for k, v in overrides.items():
        if not hasattr(cfg, k):
            raise TypeError(f"unknown Newton option {k}")
        setattr(cfg, k, int(v) if isinstance(v, bool) else v)
    return cfg


def _report(rep, recs):
    keys = [f[0] for f in capi.IterationRecord._fields_]
    return dict(converged=bool(rep.converged), load_steps=rep.load_steps_taken,
                newton_iterations=rep.newton_iterations, cg_iterations=rep.cg_iterations,
                final_fnorm=rep.final_fnorm,
                records=[{k: getattr(recs[i], k) for k in keys} for i in range(rep.num_records)])


def newton_solve(op: MatrixFreeOperator, mg: MultigridHierarchy, u, load_step=0, time=1.0,
                 **config):
    """newton_solve (nonlinear.hpp:162-216) on device vector u (updated in place)."""
    u = _dev(u, op.size())
    cfg = newton_config(**config)
    rep = capi.SolveReport()
    recs = (capi.IterationRecord * 512)()
    check(lib().hxg_newton_solve(op.h, mg.h, ctypes.byref(cfg), _ptr(u), int(load_step),
                                 float(time), ctypes.byref(rep), recs, 512))
    out = _report(rep, recs)
    out["u"] = u
    return out


class FemProblem:
    """The configured pieces of FemProblem (problem.hpp:19-58): box mesh,
    basis on q Gauss-Legendre points, geometry, whole-face Dirichlet sets,
    traction load, operator and (lazily) the p-MG hierarchy."""

    def __init__(self, extents=(1.0, 1.0, 1.0), cells=(2, 2, 2), order=2, q=0,
                 fixed_faces=("-x",), traction_face=None, traction=(0.0, 0.0, 0.0), young=1.0,
                 poisson=0.3, geometry=True, storage="current", body_force=(0.0, 0.0, 0.0),
                 mu=None, lam=None, mg_smoothing=(1, 1)):
        self.extents, self.cells, self.order = tuple(extents), tuple(cells), order
        self.q = q or order + 1
        self.basis = build_lagrange_basis(order, self.q)
        if mu is not None:  # explicit Lame parameters (config.hpp:82-85)
            self.mu, self.lam = mu, lam
        else:
            self.mu, self.lam = lame_from_young_poisson(young, poisson)
        self.mg_smoothing = tuple(mg_smoothing)
        self.mask, self.fixed_face_mask = constraint_mask(cells, order, fixed_faces)
        dx = w = None
        if geometry is True:  # host restatement of compute_geometric_factors
            dx, w = geometric_factors(extents, cells, order, self.q)
        self.op = MatrixFreeOperator(cells, self.basis, dx, w, self.mu, self.lam, self.mask,
                                     extents=extents if geometry == "box" else None,
                                     storage=storage)
        self.load = None
        if traction_face is not None:  # assemble_traction_load (operator.hpp:381-443)
            self.load = traction_load(extents, cells, order, self.q, traction_face, traction)
        if any(b != 0.0 for b in body_force):  # assemble_body_force_load (operator.hpp:440-456)
            bf = body_force_load(extents, cells, self.basis, body_force)
            self.load = bf if self.load is None else self.load + bf
        self.op.set_external_load(self.load)
        self.num_elements = cells[0] * cells[1] * cells[2]
        self.nq = self.q**3
        self._mg = None

    def size(self):
        return self.op.size()

    def solve(self, max_bisections=3, **config):
        """FemProblem::solve (problem.hpp:118-127): Newton with load
        continuation from u = 0; returns the report with the solution u."""
        u = torch.zeros(self.size(), dtype=torch.float64, device="cuda")
        cfg = newton_config(**config)
        rep = capi.SolveReport()
        recs = (capi.IterationRecord * 2048)()
        check(lib().hxg_solve_continuation(self.op.h, self.hierarchy.h, ctypes.byref(cfg),
                                           _ptr(u), int(max_bisections), ctypes.byref(rep),
                                           recs, 2048))
        out = _report(rep, recs)
        out["u"] = u
        return out

    @property
    def hierarchy(self) -> MultigridHierarchy:
        if self._mg is None:
            self._mg = MultigridHierarchy(self.op, self.fixed_face_mask,
                                          pre_smooth=self.mg_smoothing[0],
                                          post_smooth=self.mg_smoothing[1])
        return self._mg
