"""ctypes binding of the C-ABI in include/hexmg_b200.h (the drop-in boundary).

This is the Python-side equivalent of the ctypes stub shown in
INTEGRATION.md; it loads the in-tree ``libhexmg_b200.so`` and fails loudly if
it is absent.  No torch types cross the boundary: device buffers are passed as
raw pointers.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
library_path = os.environ.get("HXG_LIBRARY", os.path.join(_HERE, "libhexmg_b200.so"))

HXG_OK = 0
ERR_GENERIC = 1
ERR_INVERTED_ELEMENT = 2
ERR_STATE_NOT_INITIALIZED = 3
ERR_INDEFINITE = 4
ERR_NOT_SPD = 5
ERR_INVALID_SMOOTHER = 6
ERR_INVALID_ARGUMENT = 7
ERR_CUDA = 8
ERR_UNSUPPORTED = 9
ERR_STEP_REJECTED = 10


class HxgErrorStruct(ctypes.Structure):
    _fields_ = [("code", ctypes.c_int), ("element", ctypes.c_int), ("point", ctypes.c_int),
                ("jacobian", ctypes.c_double), ("message", ctypes.c_char * 512)]


class HxgError(RuntimeError):
    """Mirror of the reference's typed exceptions (errors.hpp:9-104)."""

    def __init__(self, code, message, element=-1, point=-1, jacobian=0.0):
        super().__init__(f"[hxg {code}] {message}")
        self.code, self.element, self.point, self.jacobian = code, element, point, jacobian


class InvertedElementError(HxgError):
    pass


class StateNotInitializedError(HxgError):
    pass


class IndefiniteOperatorError(HxgError):
    pass


class NotSpdError(HxgError):
    pass


class InvalidSmootherError(HxgError):
    pass


class StepRejectedError(HxgError):
    pass


_CLASSES = {ERR_INVERTED_ELEMENT: InvertedElementError,
            ERR_STATE_NOT_INITIALIZED: StateNotInitializedError,
            ERR_INDEFINITE: IndefiniteOperatorError, ERR_NOT_SPD: NotSpdError,
            ERR_INVALID_SMOOTHER: InvalidSmootherError, ERR_STEP_REJECTED: StepRejectedError}


class CgReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("converged", ctypes.c_int),
                ("eig_min", ctypes.c_double), ("eig_max", ctypes.c_double),
                ("initial_natural_norm", ctypes.c_double), ("final_natural_norm", ctypes.c_double)]


class NewtonConfig(ctypes.Structure):
    """NewtonConfig (nonlinear.hpp:16-24) + the line-search quirk switch."""
    _fields_ = [("max_iterations", ctypes.c_int), ("rtol", ctypes.c_double),
                ("atol", ctypes.c_double), ("linear_rtol", ctypes.c_double),
                ("linear_max_iterations", ctypes.c_int), ("use_line_search", ctypes.c_int),
                ("load_steps", ctypes.c_int), ("reference_line_search_quirk", ctypes.c_int),
                ("solver", ctypes.c_int), ("lbfgs_memory", ctypes.c_int),
                ("precond_refresh", ctypes.c_int)]


class IterationRecord(ctypes.Structure):
    """IterationRecord (nonlinear.hpp:26-36)."""
    _fields_ = [("load_step", ctypes.c_int), ("time", ctypes.c_double),
                ("iteration", ctypes.c_int), ("fnorm", ctypes.c_double),
                ("fnorm_rel", ctypes.c_double), ("cg_iterations", ctypes.c_int),
                ("cg_converged", ctypes.c_int), ("condition_estimate", ctypes.c_double),
                ("alpha", ctypes.c_double)]


class SolveReport(ctypes.Structure):
    _fields_ = [("converged", ctypes.c_int), ("load_steps_taken", ctypes.c_int),
                ("newton_iterations", ctypes.c_int), ("cg_iterations", ctypes.c_int),
                ("final_fnorm", ctypes.c_double), ("num_records", ctypes.c_int)]


class OpDesc(ctypes.Structure):
    _fields_ = [("order", ctypes.c_int), ("qpts", ctypes.c_int), ("cells", ctypes.c_int * 3),
                ("interp", ctypes.c_void_p), ("deriv", ctypes.c_void_p),
                ("colloc", ctypes.c_void_p), ("dxidX", ctypes.c_void_p),
                ("weight", ctypes.c_void_p), ("mu", ctypes.c_double),
                ("lam", ctypes.c_double), ("storage", ctypes.c_int), ("mask", ctypes.c_void_p),
                ("extents", ctypes.c_void_p), ("qweights", ctypes.c_void_p)]


# name -> argtypes (all return int unless listed in _RESTYPE)
_vp, _i, _d, _i64, _sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64, ctypes.c_size_t
_P = ctypes.POINTER
SIGNATURES = {
    "hxg_last_error": [_vp],
    "hxg_version": [],
    "hxg_state_create": [_vp],
    "hxg_state_release": [_vp],
    "hxg_op_create": [_vp, _vp, _vp],
    "hxg_op_destroy": [_vp],
    "hxg_op_size": [_vp, _P(_i64)],
    "hxg_op_num_elements": [_vp, _P(_i64)],
    "hxg_op_set_stream": [_vp, _vp],
    "hxg_op_set_external_load": [_vp, _vp],
    "hxg_op_set_load_scale": [_vp, _d],
    "hxg_op_set_jacobian_perturbation": [_vp, _d],
    "hxg_op_stored_bytes_per_dof": [_vp, _P(_d)],
    "hxg_op_counters": [_vp, _P(_i64), _P(_i64)],
    "hxg_op_apply_residual": [_vp, _vp, _vp],
    "hxg_op_apply_jacobian": [_vp, _vp, _vp],
    "hxg_op_apply_jacobian_host": [_vp, _vp, _vp],
    "hxg_op_apply_residual_host": [_vp, _vp, _vp],
    "hxg_op_extract_diagonal": [_vp, _vp],
    "hxg_op_total_strain_energy": [_vp, _vp, _P(_d)],
    "hxg_op_export_state": [_vp, _vp],
    "hxg_op_set_variant": [_vp, _i],
    "hxg_op_kernel_launches": [_vp, _P(_i)],
    "hxg_op_gather": [_vp, _vp, _vp],
    "hxg_op_scatter_add": [_vp, _vp, _vp],
    "hxg_mg_create": [_vp, _i, _vp, _i, _i, _i, _vp],
    "hxg_mg_destroy": [_vp],
    "hxg_mg_num_levels": [_vp, _P(_i)],
    "hxg_mg_level_size": [_vp, _i, _P(_i64)],
    "hxg_mg_level_op": [_vp, _i, _vp],
    "hxg_mg_setup_numeric": [_vp],
    "hxg_mg_set_coarse_mode": [_vp, _i],
    "hxg_mg_lambda_max": [_vp, _i, _P(_d)],
    "hxg_mg_prolong": [_vp, _i, _vp, _vp],
    "hxg_mg_restrict": [_vp, _i, _vp, _vp],
    "hxg_mg_vcycle": [_vp, _vp, _vp],
    "hxg_mg_smooth": [_vp, _i, _vp, _vp],
    "hxg_mg_coarse_nnz": [_vp, _P(_i64)],
    "hxg_mg_coarse_csr_host": [_vp, _vp, _vp, _vp],
    "hxg_mg_hmg_levels": [_vp, _P(_i)],
    "hxg_mg_hmg_level_nnz": [_vp, _i, _P(_i64), _P(_i64)],
    "hxg_mg_hmg_level_csr_host": [_vp, _i, _vp, _vp, _vp, _vp],
    "hxg_mg_coarse_solve": [_vp, _vp, _vp],
    "hxg_mg_assemble_coarse": [_vp],
    "hxg_chol_create": [_i, _vp, _vp, _vp, _i, _vp],
    "hxg_chol_factorize": [_vp, _vp],
    "hxg_chol_factorize_device": [_vp, _vp],
    "hxg_asm_create": [_vp, _vp],
    "hxg_asm_numeric": [_vp],
    "hxg_asm_nnz": [_vp, _vp],
    "hxg_asm_matvec": [_vp, _vp, _vp],
    "hxg_asm_csr_host": [_vp, _vp, _vp, _vp],
    "hxg_asm_destroy": [_vp],
    "hxg_mg_coarse_vals_device": [_vp, _vp],
    "hxg_chol_solve": [_vp, _vp, _vp],
    "hxg_chol_destroy": [_vp],
    "hxg_cg_solve": [_vp, _vp, _i, _vp, _vp, _d, _i, _vp, _vp, _i],
    "hxg_lambda_max_jacobi": [_vp, _i, _P(_d)],
    "hxg_newton_config_default": [_vp],
    "hxg_newton_solve": [_vp, _vp, _vp, _vp, _i, _d, _vp, _vp, _i],
    "hxg_lbfgs_solve": [_vp, _vp, _vp, _vp, _i, _d, _vp, _vp, _i],
    "hxg_solve_continuation": [_vp, _vp, _vp, _vp, _i, _vp, _vp, _i],
    "hxg_dot": [_vp, _vp, _i64, _vp, _P(_d)],
    "hxg_malloc": [_vp, _sz],
    "hxg_free": [_vp],
    "hxg_pointer_is_device": [_vp, _vp],
    "hxg_comm_create": [_i, _i, _vp, _vp],
    "hxg_nccl_unique_id": [_vp],
    "hxg_comm_create_nccl": [_i, _i, _vp, _vp],
    "hxg_comm_destroy": [_vp],
    "hxg_partition_block": [_vp, _vp, _i, _vp, _vp],
    "hxg_mg_create_partitioned": [_vp, _vp, _vp, _vp, _i, _vp, _i, _i, _i, _vp],
    "hxg_mg_apply": [_vp, _i, _vp, _vp],
    "hxg_mg_dot": [_vp, _i, _vp, _vp, _vp],
    "hxg_mg_residual": [_vp, _vp, _vp],
    "hxg_stream_synchronize": [_vp],
    "hxg_memcpy_h2d": [_vp, _vp, _sz],
    "hxg_memcpy_d2h": [_vp, _vp, _sz],
    "hxg_device_synchronize": [],
    "hxg_setup_basis": [_i, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "hxg_setup_geometry": [_vp, _vp, _i, _i, _vp, _vp],
    "hxg_setup_constraints": [_vp, _i, _i, _vp],
    "hxg_setup_traction_load": [_vp, _vp, _i, _i, _i, _vp, _vp],
    "hxg_op_time_jacobian": [_vp, _vp, _vp, _i, _i, _P(_d)],
    "hxg_op_time_jacobian_parts": [_vp, _vp, _vp, _i, _i, _vp],
}
_RESTYPE = {"hxg_version": ctypes.c_char_p}

_lib = None


def lib():
    """Load the CUDA library (raises if it was not built — no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(library_path):
            raise ImportError(
                f"{library_path} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(library_path)
        for name, args in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = _RESTYPE.get(name, ctypes.c_int)
        _lib = L
    return _lib


def check(rc):
    if rc != HXG_OK:
        e = HxgErrorStruct()
        lib().hxg_last_error(ctypes.byref(e))
        cls = _CLASSES.get(rc, HxgError)
        raise cls(rc, e.message.decode(errors="replace"), e.element, e.point, e.jacobian)
