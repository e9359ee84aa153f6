"""ctypes binding of libsgiga.so (the C ABI declared in include/sgiga.h).

The product path has no CPU fallback: if the shared object is missing or
cannot find a CUDA device, every entry point raises.
"""
from __future__ import annotations

import ctypes as ct
import threading
from pathlib import Path

import numpy as np

from .errors import DeviceError, EmptyInteriorError, InvalidGeometryError, LinearSolveError

LIB_PATH = Path(__file__).resolve().with_name("libsgiga.so")

SGIGA_OK = 0
SGIGA_ERR_VALUE = -1
SGIGA_ERR_GEOMETRY = -2
SGIGA_ERR_SOLVE = -3
SGIGA_ERR_EMPTY = -4
SGIGA_ERR_CUDA = -5
SGIGA_ERR_STATE = -6
SGIGA_ERR_KEY = -7

FLAG_ASSEMBLY_ONLY = 1   # sgiga_flags

FORCING_HOST = -1
FORCING_ZERO = 0
FORCING_SIN_PRODUCT = 1
FORCING_ANNULUS_POLAR = 2
FORCING_EXP_BUBBLE = 3
FORCING_CUBE_POLY = 4
FORCING_ANNULUS_2D = 5
FORCING_ANNULUS_3D = 6
FORCING_CONSTANT_ONE = 7
FORCING_LSHAPE = 8

# every symbol include/sgiga.h declares (checked by tests/test_boundary.py)
EXPORTED = (
    "sgiga_create", "sgiga_upload", "sgiga_batch_sizes", "sgiga_quad_points_physical",
    "sgiga_set_forcing_density", "sgiga_component_info", "sgiga_assemble", "sgiga_solve",
    "sgiga_coefficients", "sgiga_set_coefficients", "sgiga_combine_points", "sgiga_run",
    "sgiga_run_async", "sgiga_run_wait", "sgiga_run_host_async",
    "sgiga_combine_grid", "sgiga_error_norms", "sgiga_subset_error_norms", "sgiga_export_csr", "sgiga_phase_stats",
    "sgiga_basis_table", "sgiga_plan_order_sum", "sgiga_run_components_async", "sgiga_edge_projection_batch",
    "sgiga_iterations", "sgiga_kernel_times", "sgiga_stream", "sgiga_destroy", "sgiga_last_error",
    "sgiga_device_count", "sgiga_local_poisson_systems",
    "sgiga_full_patch_system", "sgiga_edge_projection_system", "sgiga_gather_sum", "sgiga_gather",
    "sgiga_csr_spmv_sub", "sgiga_csr_pcg", "sgiga_set_coefficients_device", "sgiga_assembly_flops",
    "sgiga_assembly_kind",
)


class ProblemDesc(ct.Structure):
    """struct sgiga_problem_desc (include/sgiga.h)."""

    _fields_ = [
        ("d", ct.c_int32),
        ("degree", ct.c_int32),
        ("regularity", ct.c_int32),
        ("quad_points", ct.c_int32),
        ("n_comp", ct.c_int32),
        ("levels", ct.POINTER(ct.c_int32)),
        ("coefs", ct.POINTER(ct.c_int32)),
        ("gauss_nodes", ct.POINTER(ct.c_double)),
        ("gauss_weights", ct.POINTER(ct.c_double)),
        ("max_level", ct.c_int32),
        ("bp_offset", ct.POINTER(ct.c_int64)),
        ("bp_count", ct.POINTER(ct.c_int32)),
        ("breakpoints", ct.POINTER(ct.c_double)),
        ("geo_degree", ct.POINTER(ct.c_int32)),
        ("geo_nknots", ct.POINTER(ct.c_int32)),
        ("geo_knots", ct.POINTER(ct.c_double)),
        ("geo_hw", ct.POINTER(ct.c_double)),
        ("forcing_id", ct.c_int32),
        ("flags", ct.c_int32),
    ]


_lock = threading.Lock()
_lib = None

P_I32 = ct.POINTER(ct.c_int32)
P_I64 = ct.POINTER(ct.c_int64)
P_F64 = ct.POINTER(ct.c_double)
P_F32 = ct.POINTER(ct.c_float)
VP = ct.c_void_p


def _declare(lib):
    sig = {
        "sgiga_create": ([ct.POINTER(ProblemDesc), VP, ct.POINTER(VP)], ct.c_int),
        "sgiga_upload": ([VP, ct.POINTER(ProblemDesc)], ct.c_int),
        "sgiga_batch_sizes": ([VP, P_I64, P_I64, P_I64, P_I64], ct.c_int),
        "sgiga_quad_points_physical": ([VP, P_F64], ct.c_int),
        "sgiga_set_forcing_density": ([VP, P_F64], ct.c_int),
        "sgiga_component_info": ([VP, P_I32, P_I64], ct.c_int),
        "sgiga_assemble": ([VP], ct.c_int),
        "sgiga_solve": ([VP, ct.c_double, ct.c_int32, P_I32, P_F64], ct.c_int),
        "sgiga_coefficients": ([VP, P_F64], ct.c_int),
        "sgiga_set_coefficients": ([VP, P_F64], ct.c_int),
        "sgiga_combine_points": ([VP, VP, ct.c_int64, VP, ct.c_int32], ct.c_int),
        "sgiga_run": ([VP, ct.c_double, ct.c_int32, VP, ct.c_int64, VP, ct.c_int32, P_I32, P_F64], ct.c_int),
        "sgiga_run_async": ([VP, ct.c_double, ct.c_int32, VP, ct.c_int64, VP], ct.c_int),
        "sgiga_run_wait": ([VP, P_I32, P_F64], ct.c_int),
        "sgiga_run_host_async": ([VP, ct.c_double, ct.c_int32, VP, ct.c_int64, VP], ct.c_int),
        "sgiga_combine_grid": ([VP, P_F64, P_I64, ct.c_int32, P_F64, P_F64], ct.c_int),
        "sgiga_error_norms": ([VP, P_F64, P_F64, P_I64, ct.c_int32, P_F64], ct.c_int),
        "sgiga_subset_error_norms": ([VP, P_F64, P_F64, P_I64, ct.c_int32, P_I32, P_F64, ct.c_int32, P_F64], ct.c_int),
        "sgiga_full_patch_system": ([VP, ct.c_int32, VP, VP], ct.c_int),
        "sgiga_edge_projection_system": ([VP, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, VP, VP], ct.c_int),
        "sgiga_gather_sum": ([VP, ct.c_int64, VP, VP, VP, VP], ct.c_int),
        "sgiga_gather": ([VP, ct.c_int64, VP, VP, VP], ct.c_int),
        "sgiga_csr_spmv_sub": ([VP, ct.c_int64, VP, VP, VP, VP, VP], ct.c_int),
        "sgiga_csr_pcg": ([VP, ct.c_int32, VP, ct.c_int64, VP, VP, VP, VP, VP, ct.c_double, ct.c_int32,
                           P_I32, P_F64], ct.c_int),
        "sgiga_set_coefficients_device": ([VP, VP], ct.c_int),
        "sgiga_export_csr": ([VP, ct.c_int32, P_I64, P_I64, P_I32, P_F64, P_F64], ct.c_int),
        "sgiga_phase_stats": ([VP, P_F32, P_I64], ct.c_int),
        "sgiga_run_components_async": ([VP, ct.c_double, ct.c_int32, VP, ct.c_int64, VP], ct.c_int),
        "sgiga_edge_projection_batch": ([VP, ct.c_int32, VP, VP, ct.c_int32, ct.c_int32, VP], ct.c_int),
        "sgiga_plan_order_sum": ([VP, ct.c_int32, ct.c_int64, VP, VP, VP, VP], ct.c_int),
        "sgiga_basis_table": ([VP, ct.c_int32, ct.c_int32, P_I32, P_F64, P_F64, P_F64, P_F64], ct.c_int),
        "sgiga_iterations": ([VP, P_I32], ct.c_int),
        "sgiga_kernel_times": ([VP, P_F32], ct.c_int),
        "sgiga_assembly_flops": ([VP, P_F64], ct.c_int),
        "sgiga_assembly_kind": ([VP, P_I32], ct.c_int),
        "sgiga_stream": ([VP], VP),
        "sgiga_destroy": ([VP], ct.c_int),
        "sgiga_last_error": ([], ct.c_char_p),
        "sgiga_device_count": ([P_I32], ct.c_int),
        "sgiga_local_poisson_systems": (
            [ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int32, ct.c_int64, ct.c_int32, ct.c_int32,
             P_F64, P_F64, P_I64, P_I32, P_I32, P_F64, P_F64, P_F64, P_F64], ct.c_int),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res


def load():
    """Load libsgiga.so once; raises if it is missing (no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is not built; run `python -m paper_1707_09598_b200.build` "
                    "(the GPU path has no CPU fallback)"
                )
            lib = ct.CDLL(str(LIB_PATH))
            _declare(lib)
            _lib = lib
    return _lib


def last_error() -> str:
    msg = load().sgiga_last_error()
    return msg.decode() if msg else ""


def check(code: int):
    """Map a status code to the reference's exception classes."""
    if code == SGIGA_OK:
        return
    msg = last_error()
    if code == SGIGA_ERR_GEOMETRY:
        raise InvalidGeometryError(msg)
    if code == SGIGA_ERR_SOLVE:
        raise LinearSolveError(msg)
    if code == SGIGA_ERR_EMPTY:
        raise EmptyInteriorError(msg)
    if code == SGIGA_ERR_KEY:
        raise KeyError(msg)
    if code == SGIGA_ERR_CUDA:
        raise DeviceError(msg)
    if code == SGIGA_ERR_STATE:
        raise RuntimeError(msg)
    raise ValueError(msg)


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(ct.POINTER(ctype))


def device_count() -> int:
    n = ct.c_int32(0)
    load().sgiga_device_count(ct.byref(n))
    return int(n.value)
