"""ctypes binding of libddpma.so (include/ddpma.h).

The library is built in-tree (``make`` / ``__graft_entry__.build()``).  There
is no CPU fallback: if the shared object is missing every entry point raises
:class:`DdmeshError` — loudly — instead of silently computing elsewhere.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import (ConfigurationError, DdmeshError, InvalidMonitorError,
                     StiffnessError)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DDPMA_LIB") or os.path.join(_HERE, "libddpma.so")

OK, ERR_CONFIG, ERR_INVALID_MONITOR, ERR_STIFFNESS, ERR_CUDA, ERR_STATE, ERR_VALUE, \
    ERR_OVERFLOW, ERR_IO = range(9)
FACE_PHYSICAL, FACE_INTERFACE = 0, 1
ALTERNATING, PARALLEL = 0, 1
STOP_MIN, STOP_MAX = 0, 1
SCHEME_ADAPTIVE, SCHEME_EULER = 0, 1
MON_UNIFORM, MON_RING, MON_MIXTURE = 0, 1, 2
MON_BURGERS2D, MON_SPIRAL2D, MON_SPHERE3D, MON_NINE_SPHERES3D, MON_QUASI1D_LINEAR = 3, 4, 5, 6, 7
MON_SAMPLED = 8
NCLASS = 3   # profiling classes: 0 eval (window kernel), 1 mesh/density, 2 other


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int), ("counts", C.c_int * 3),
                ("extents", (C.c_double * 2) * 3), ("explicit_geom", C.c_int),
                ("spacing", C.c_double * 3), ("measure", C.c_double),
                ("face_coord", (C.c_double * 2) * 3)]


class Subdomain(C.Structure):
    _fields_ = [("id", C.c_int), ("pos", C.c_int * 3), ("box", (C.c_int * 2) * 3),
                ("owned", (C.c_int * 2) * 3), ("face", (C.c_int * 2) * 3),
                ("donor", (C.c_int * 2) * 3)]


class Monitor(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", C.c_int), ("domain", (C.c_double * 2) * 3),
                ("constant", C.c_double), ("center", C.c_double * 3),
                ("amp", C.c_double), ("sharp", C.c_double), ("r2", C.c_double),
                ("nbumps", C.c_int), ("c", C.POINTER(C.c_double)),
                ("s", C.POINTER(C.c_double)), ("a", C.POINTER(C.c_double)),
                ("eps", C.c_double), ("u_backed", C.c_int),
                ("lat", C.c_int * 3), ("axes", C.POINTER(C.c_double) * 3),
                ("values", C.POINTER(C.c_double)), ("grads", C.POINTER(C.c_double) * 3)]


class SolverCfg(C.Structure):
    _fields_ = [("dtau", C.c_double), ("tol", C.c_double), ("transmission", C.c_int),
                ("stop_rule", C.c_int), ("max_windows", C.c_int), ("scheme", C.c_int),
                ("substeps", C.c_int), ("rtol", C.c_double), ("atol", C.c_double),
                ("max_stages", C.c_int), ("det_floor", C.c_double),
                ("monitor_smooth_passes", C.c_int), ("monitor_relax", C.c_double)]


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_I64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); every symbol include/ddpma.h declares.
SIGNATURES = {
    "ddpma_global_error": (C.c_char_p, []),
    "ddpma_build_decomposition": (C.c_int, [C.c_int, _I, _I, C.c_int, C.POINTER(Subdomain),
                                            C.c_int, _I]),
    "ddpma_rkc_coeffs": (C.c_int, [C.c_int, _D, _D, _D, _D, _D, _D, _D]),
    "ddpma_plan_create": (C.c_int, [C.POINTER(Grid), C.POINTER(Subdomain), C.c_int, _I,
                                    C.c_int, C.POINTER(Monitor), C.POINTER(SolverCfg),
                                    C.c_int, C.POINTER(_P)]),
    "ddpma_plan_destroy": (None, [_P]),
    "ddpma_last_error": (C.c_char_p, [_P]),
    "ddpma_set_state": (C.c_int, [_P, _D]),
    "ddpma_run": (C.c_int, [_P, C.c_int, C.c_double, _D, _D, _I, _I, _D]),
    "ddpma_error_info": (C.c_int, [_P, _I, _D, _D, _I64]),
    "ddpma_error_nodes": (C.c_int, [_P, _I64, C.c_int64]),
    "ddpma_assemble_dev": (C.c_int, [_P, C.c_void_p, C.c_void_p, C.c_void_p]),
    "ddpma_assemble_host": (C.c_int, [_P, _D, _D, _D]),
    "ddpma_get_sub_psi": (C.c_int, [_P, C.c_int, _D]),
    "ddpma_overlap_gap": (C.c_int, [_P, _D]),
    "ddpma_density": (C.c_int, [_P, _D, _D, _D, _D, _D]),
    "ddpma_begin_window": (C.c_int, [_P, C.c_double, C.c_double]),
    "ddpma_trace_counts": (C.c_int, [_P, _I, C.c_int, C.c_int, _I64, _I64]),
    "ddpma_pack_traces": (C.c_int, [_P, C.c_void_p]),
    "ddpma_apply_traces": (C.c_int, [_P, C.c_void_p]),
    "ddpma_advance": (C.c_int, [_P]),
    "ddpma_rhs_frozen": (C.c_int, [_P, C.c_int, _D, _D, C.c_double, _D, _I]),
    "ddpma_mesh": (C.c_int, [_P, C.c_int, _D, _D, _D]),
    "ddpma_raw_density": (C.c_int, [_P, C.c_int, _D, _D]),
    "ddpma_residual": (C.c_int, [_P, C.c_int, _D, _D, _D]),
    "ddpma_quality": (C.c_int, [_P, C.c_int, _D, C.c_double, C.c_int, _D, _D]),
    "ddpma_relative_errors": (C.c_int, [_P, C.c_int, _D, _D, _D]),
    "ddpma_rkc_step": (C.c_int, [_P, C.c_int, _D, _D, C.c_double, C.c_double, C.c_int,
                                 _D, _D, _I, _I]),
    "ddpma_counters": (C.c_int, [_P, _I64, _I64, _I64, _D]),
    "ddpma_integrate_window": (C.c_int, [_P, C.c_int, _D, _D, C.c_double]),
    "ddpma_pack_owned": (C.c_int, [_P, C.c_void_p, _I64]),
    "ddpma_sub_evals": (C.c_int, [_P, _I64, C.c_int]),
    "ddpma_set_profiling": (C.c_int, [_P, C.c_int]),
    "ddpma_profile": (C.c_int, [_P, _D, _D, _I64, _I64, C.c_int]),
    "ddpma_alternating_levels": (C.c_int, [C.c_int, C.POINTER(Subdomain), C.c_int, _I]),
    "ddpma_stream": (C.c_void_p, [_P]),
    "ddpma_window_kernel": (C.c_char_p, [_P]),
    "ddpma_monitor_mass": (C.c_int, [C.POINTER(Monitor), _I, C.c_int, _D, _D, _I]),
    "ddpma_write_mesh_vtk": (C.c_int, [C.c_char_p, C.c_int, _I, _D, _D, _D, C.c_char_p,
                                       C.c_char_p]),
    "ddpma_io_error": (C.c_char_p, []),
}

_lib = None


def lib():
    """Load libddpma.so once; raise DdmeshError if it is absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DdmeshError(
                f"libddpma.so not built at {LIB_PATH}: run `make` (or "
                "__graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def dptr(a: np.ndarray):
    return a.ctypes.data_as(_D)


def raise_status(st: int, msg: str):
    if st == OK:
        return
    if st == ERR_CONFIG:
        raise ConfigurationError(msg)
    if st == ERR_INVALID_MONITOR:
        raise InvalidMonitorError(msg)
    if st == ERR_STIFFNESS:
        raise StiffnessError(msg)
    if st == ERR_VALUE:
        raise ValueError(msg)
    if st == ERR_IO:
        raise OSError(msg)
    if st == ERR_OVERFLOW:
        raise OverflowError(msg)
    raise DdmeshError(msg)


def check_global(st: int):
    if st != OK:
        raise_status(st, lib().ddpma_global_error().decode())


def require_cuda():
    """The compute entry points need a CUDA device; fail loudly without one."""
    try:
        import torch
        ok = torch.cuda.is_available()
    except Exception:  # pragma: no cover - torch is part of the image
        ok = False
    if not ok:
        raise DdmeshError("no CUDA device: the DDPMA solver runs only on the GPU "
                          "(there is no CPU fallback)")
