"""ORACLE / TEST INFRASTRUCTURE ONLY — ctypes handle on oracle/_ref/libhexmg_ref.so,
the unmodified reference headers compiled by oracle/Makefile (see ref_driver.cpp
for the reference call behind each entry point).  Used by tests/, smoke() and
bench.py's CPU-baseline leg only."""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libhexmg_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(LIB_PATH)
        vp, i, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_create.restype = vp
        L.ref_create.argtypes = [vp, vp, i, i, i, i, vp, d, d, i]
        L.ref_destroy.argtypes = [vp]
        for name in ("ref_size", "ref_num_elements", "ref_points_per_element", "ref_num_levels",
                     "ref_coarse_nnz"):
            getattr(L, name).argtypes = [vp]
        L.ref_level_size.argtypes = [vp, i]
        L.ref_level_order.argtypes = [vp, i]
        L.ref_set_threads.argtypes = [vp, i]
        L.ref_set_time.argtypes = [vp, d]
        L.ref_set_jacobian_perturbation.argtypes = [vp, d]
        L.ref_basis.argtypes = [i, i] + [vp] * 7
        L.ref_mesh_coords.argtypes = [vp, vp]
        L.ref_restriction.argtypes = [vp, i, vp, vp]
        L.ref_geometry.argtypes = [vp, vp, vp]
        L.ref_constraints.argtypes = [vp, i, vp, vp]
        L.ref_external_load.argtypes = [vp, vp]
        L.ref_impose_dirichlet.argtypes = [vp, vp]
        L.ref_apply_residual.argtypes = [vp, vp, vp]
        L.ref_apply_jacobian.argtypes = [vp, i, vp, vp]
        L.ref_extract_diagonal.argtypes = [vp, i, vp]
        L.ref_state.argtypes = [vp, vp]
        L.ref_set_storage.argtypes = [i]
        L.ref_state_stride.argtypes = [vp]
        L.ref_energy.argtypes = [vp, vp, vp]
        L.ref_stored_bytes_per_dof.argtypes = [vp]
        L.ref_stored_bytes_per_dof.restype = d
        L.ref_mg_setup.argtypes = [vp]
        L.ref_level_lambda_max.argtypes = [vp, i]
        L.ref_level_lambda_max.restype = d
        L.ref_level_inv_diag.argtypes = [vp, i, vp]
        L.ref_prolong.argtypes = [vp, i, vp, vp]
        L.ref_restrict.argtypes = [vp, i, vp, vp]
        L.ref_smoother_apply.argtypes = [vp, i, vp, vp]
        L.ref_vcycle.argtypes = [vp, vp, vp]
        L.ref_coarse_csr.argtypes = [vp, vp, vp, vp]
        L.ref_cg.argtypes = [vp, i, vp, vp, d, i, vp, vp, vp, vp, vp, i]
        L.ref_lambda_max_jacobi.argtypes = [vp, i, i, vp]
        L.ref_rough_seed.argtypes = [i, vp, vp]
        L.ref_time_jacobian.argtypes = [vp, vp, i, i]
        L.ref_time_jacobian.restype = d
        L.ref_newton.argtypes = [vp, i, i, d, vp, vp, vp, vp]
        L.ref_solve.argtypes = [vp, i, i, d, i, i, i, vp, vp, vp, vp]
        L.ref_verify.argtypes = [i, d, vp, i]
        L.ref_write_vtk.argtypes = [vp, vp, vp, i]
        for name in ("ref_parse_config", "ref_accuracy_study", "ref_performance_study"):
            getattr(L, name).argtypes = [ctypes.c_char_p, vp, i]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


FACES = {"-x": 0, "+x": 1, "-y": 2, "+y": 3, "-z": 4, "+z": 5}


def basis(p, q):
    L = lib()
    n = p + 1
    out = dict(nodes=np.zeros(n), points=np.zeros(q), weights=np.zeros(q), interp=np.zeros((q, n)),
               deriv=np.zeros((q, n)), pinv=np.zeros((n, q)), colloc=np.zeros((q, q)))
    _check(L.ref_basis(p, q, *[_p(out[k]) for k in
                               ("nodes", "points", "weights", "interp", "deriv", "pinv", "colloc")]))
    return out


class RefProblem:
    """FemProblem (problem.hpp:19-58) built by the reference itself."""

    def __init__(self, extents=(1.0, 1.0, 1.0), cells=(2, 2, 2), order=2, q=0, fixed=("-x",),
                 traction_face=None, traction=(0.0, 0.0, 0.0), young=1.0, poisson=0.3, threads=1,
                 storage=0):
        L = lib()
        L.ref_set_storage(storage)
        ext = np.asarray(extents, dtype=np.float64)
        cl = np.asarray(cells, dtype=np.int32)
        tr = np.asarray(traction, dtype=np.float64)
        mask = 0
        for f in fixed:
            mask |= 1 << FACES[f]
        tf = -1 if traction_face is None else FACES[traction_face]
        h = L.ref_create(_p(ext), _p(cl), order, q, mask, tf, _p(tr), young, poisson, threads)
        L.ref_set_storage(0)
        if not h:
            raise RefError(-1, L.ref_last_error().decode())
        self.h = ctypes.c_void_p(h)
        self.order, self.q = order, (q or order + 1)
        self.extents, self.cells = tuple(extents), tuple(cells)
        self.n = L.ref_size(self.h)
        self.E = L.ref_num_elements(self.h)
        self.nq = L.ref_points_per_element(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_destroy(self.h)
            self.h = None

    @property
    def num_levels(self):
        return lib().ref_num_levels(self.h)

    def level_size(self, k):
        return lib().ref_level_size(self.h, k)

    def level_order(self, k):
        return lib().ref_level_order(self.h, k)

    def set_threads(self, t):
        lib().ref_set_threads(self.h, t)

    def set_time(self, t):
        lib().ref_set_time(self.h, t)

    def write_vtk(self, u, cap=1 << 24):
        """write_vtk (vtk.hpp:15-55) of u on this problem's mesh, as text."""
        buf = ctypes.create_string_buffer(cap)
        u = np.ascontiguousarray(u, np.float64)
        _check(lib().ref_write_vtk(self.h, _p(u), ctypes.cast(buf, ctypes.c_void_p), cap))
        return buf.value.decode()

    def coords(self):
        out = np.zeros(self.n)
        lib().ref_mesh_coords(self.h, _p(out))
        return out.reshape(-1, 3)

    def restriction(self, level=-1):
        n = self.n if level < 0 else self.level_size(level)
        order = self.order if level < 0 else self.level_order(level)
        idx = np.zeros((self.E, (order + 1) ** 3), dtype=np.int32)
        mult = np.zeros(n // 3, dtype=np.int32)
        lib().ref_restriction(self.h, level, _p(idx), _p(mult))
        return idx, mult

    def geometry(self):
        dx = np.zeros((self.E, self.nq, 3, 3))
        w = np.zeros((self.E, self.nq))
        lib().ref_geometry(self.h, _p(dx), _p(w))
        return dx, w

    def constraints(self, level=-1):
        n = self.n if level < 0 else self.level_size(level)
        m = np.zeros(n, dtype=np.uint8)
        v = np.zeros(n)
        lib().ref_constraints(self.h, level, _p(m), _p(v))
        return m, v

    def external_load(self):
        out = np.zeros(self.n)
        lib().ref_external_load(self.h, _p(out))
        return out

    def impose_dirichlet(self, u):
        lib().ref_impose_dirichlet(self.h, _p(u))
        return u

    def apply_residual(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        f = np.zeros(self.n)
        _check(lib().ref_apply_residual(self.h, _p(u), _p(f)))
        return f

    def apply_jacobian(self, du, level=-1):
        n = self.n if level < 0 else self.level_size(level)
        du = np.ascontiguousarray(du, dtype=np.float64)
        y = np.zeros(n)
        _check(lib().ref_apply_jacobian(self.h, level, _p(du), _p(y)))
        return y

    def extract_diagonal(self, level=-1):
        n = self.n if level < 0 else self.level_size(level)
        d = np.zeros(n)
        _check(lib().ref_extract_diagonal(self.h, level, _p(d)))
        return d

    def state(self):
        out = np.zeros((self.E, self.nq, lib().ref_state_stride(self.h)))
        lib().ref_state(self.h, _p(out))
        return out

    def energy(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        out = ctypes.c_double()
        _check(lib().ref_energy(self.h, _p(u), ctypes.byref(out)))
        return out.value

    def stored_bytes_per_dof(self):
        return lib().ref_stored_bytes_per_dof(self.h)

    def mg_setup(self):
        _check(lib().ref_mg_setup(self.h))

    def lambda_max(self, k):
        return lib().ref_level_lambda_max(self.h, k)

    def inv_diag(self, k):
        out = np.zeros(self.level_size(k))
        lib().ref_level_inv_diag(self.h, k, _p(out))
        return out

    def prolong(self, coarse_level, xc):
        xc = np.ascontiguousarray(xc, dtype=np.float64)
        xf = np.zeros(self.level_size(coarse_level + 1))
        _check(lib().ref_prolong(self.h, coarse_level, _p(xc), _p(xf)))
        return xf

    def restrict(self, coarse_level, xf):
        xf = np.ascontiguousarray(xf, dtype=np.float64)
        xc = np.zeros(self.level_size(coarse_level))
        _check(lib().ref_restrict(self.h, coarse_level, _p(xf), _p(xc)))
        return xc

    def smoother_apply(self, k, b, x):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.array(x, dtype=np.float64)
        _check(lib().ref_smoother_apply(self.h, k, _p(b), _p(x)))
        return x

    def vcycle(self, b, x=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.n) if x is None else np.array(x, dtype=np.float64)
        _check(lib().ref_vcycle(self.h, _p(b), _p(x)))
        return x

    def coarse_csr(self):
        nnz = lib().ref_coarse_nnz(self.h)
        n = self.level_size(0)
        rp = np.zeros(n + 1, dtype=np.int32)
        cols = np.zeros(nnz, dtype=np.int32)
        vals = np.zeros(nnz)
        lib().ref_coarse_csr(self.h, _p(rp), _p(cols), _p(vals))
        return rp, cols, vals

    def cg(self, b, precond="mg", rtol=1e-8, maxit=500, x0=None):
        pc = {"none": 0, "jacobi": 1, "mg": 2}[precond]
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.zeros(self.n) if x0 is None else np.array(x0, dtype=np.float64)
        its, conv = ctypes.c_int(), ctypes.c_int()
        emin, emax = ctypes.c_double(), ctypes.c_double()
        hist = np.zeros(maxit + 2)
        _check(lib().ref_cg(self.h, pc, _p(b), _p(x), rtol, maxit, ctypes.byref(its),
                            ctypes.byref(conv), ctypes.byref(emin), ctypes.byref(emax), _p(hist),
                            maxit + 2))
        return dict(x=x, iterations=its.value, converged=bool(conv.value), eig_min=emin.value,
                    eig_max=emax.value, history=hist[: its.value + 1].copy())

    def lambda_max_jacobi(self, level=-1, iterations=10):
        out = ctypes.c_double()
        _check(lib().ref_lambda_max_jacobi(self.h, level, iterations, ctypes.byref(out)))
        return out.value

    def time_jacobian(self, x, warmup=3, repeats=20):
        x = np.ascontiguousarray(x, dtype=np.float64)
        return lib().ref_time_jacobian(self.h, _p(x), warmup, repeats)

    def newton(self, load_steps=1, line_search=False, linear_rtol=1e-3):
        u = np.zeros(self.n)
        ni, ci, fn = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        _check(lib().ref_newton(self.h, load_steps, int(line_search), linear_rtol, _p(u),
                                ctypes.byref(ni), ctypes.byref(ci), ctypes.byref(fn)))
        return dict(u=u, newton_iterations=ni.value, cg_iterations=ci.value, final_fnorm=fn.value)

    def solve(self, load_steps=1, line_search=True, linear_rtol=1e-3, solver=0, memory=5,
              refresh=0):
        """FemProblem::solve with the configured solver (0 Newton, 1 L-BFGS)."""
        u = np.zeros(self.n)
        ni, ci, fn = ctypes.c_int(), ctypes.c_int(), ctypes.c_double()
        _check(lib().ref_solve(self.h, load_steps, int(line_search), linear_rtol, solver, memory,
                               refresh, _p(u), ctypes.byref(ni), ctypes.byref(ci),
                               ctypes.byref(fn)))
        return dict(u=u, iterations=ni.value, cg_iterations=ci.value, final_fnorm=fn.value)


def rough_seed(n, mask=None):
    out = np.zeros(n)
    lib().ref_rough_seed(n, _p(mask) if mask is not None else None, _p(out))
    return out


def verify(threads=1, perturbation=0.0):
    buf = ctypes.create_string_buffer(16384)
    _check(lib().ref_verify(threads, perturbation, buf, 16384))
    out = {}
    for line in buf.value.decode().splitlines():
        name, ok, detail = line.split(":", 2)
        out[name] = (ok == "1", detail)
    return out


def _text_call(name, text, cap=1 << 20):
    buf = ctypes.create_string_buffer(cap)
    rc = getattr(lib(), name)(text.encode(), ctypes.cast(buf, ctypes.c_void_p), cap)
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())
    return buf.value.decode()


def parse_config(text):
    """parse_problem_config -> canonical 'key=value' dump (ref_driver.cpp)."""
    return _text_call("ref_parse_config", text)


def accuracy_study(text):
    """run_accuracy_study CSV for a config text."""
    return _text_call("ref_accuracy_study", text)


def performance_study(text):
    """run_performance_study CSV for a config text."""
    return _text_call("ref_performance_study", text)
