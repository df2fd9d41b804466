"""ctypes mirror of include/cisdc_gpu.h (plain C structs; no torch types cross the boundary)."""
from __future__ import annotations

import ctypes as C
import os

MAX_M = 8
MAX_SPECIES = 16
MAX_REACTIONS = 64

OK, E_INVALID_ARGUMENT, E_FACTORIZATION, E_SOLVE, E_NUMERIC, E_CAPABILITY, E_CUDA, E_IO = range(8)
PROBLEM_PERIODIC_ADR, PROBLEM_REFERENCE_RD, PROBLEM_LINEAR_SCALAR = 0, 1, 2
REACTION_NONE, REACTION_LINEAR_DECAY, REACTION_BISTABLE, REACTION_MASS_ACTION = 0, 1, 2, 3
DIFFUSION_DIRECT, DIFFUSION_MULTIGRID, DIFFUSION_BANDED_ORACLE = 0, 1, 2
FIELD_PHI, FIELD_FA, FIELD_FD, FIELD_FR, FIELD_PHI_AD = 0, 1, 2, 3, 4
STAGE_ADVECTION, STAGE_DIFFUSION, STAGE_REACTION, STAGE_COUPLED = 0, 1, 2, 3

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)


class ProblemDescC(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("ndim", C.c_int),
        ("n", C.c_int * 3),
        ("nspecies", C.c_int),
        ("h", C.c_double * 3),
        ("vel", (_dp * 3) * 3),
        ("diffusivity", _dp),
        ("reaction_kind", C.c_int),
        ("lam", C.c_double),
        ("theta", C.c_double),
        ("n_reactions", C.c_int),
        ("reactants", _ip),
        ("products", _ip),
        ("rate_constants", _dp),
        ("newton_tol", C.c_double),
        ("newton_max_iter", C.c_int),
        ("diffusion_solver", C.c_int),
        ("mg_tol", C.c_double),
        ("mg_max_cycles", C.c_int),
        ("mg_pre", C.c_int),
        ("mg_post", C.c_int),
        ("mg_coarse_sweeps", C.c_int),
        ("mg_min_coarse", C.c_int),
        ("mg_omega", C.c_double),
        ("ref_a", C.c_double),
        ("ref_d", C.c_double),
        ("ref_r", C.c_double),
        ("coupled_tol", C.c_double),
        ("coupled_max_iter", C.c_int),
    ]


class TablesC(C.Structure):
    _fields_ = [
        ("M", C.c_int),
        ("convention", C.c_int),
        ("tau", C.c_double * (MAX_M + 1)),
        ("dtau", C.c_double * MAX_M),
        ("Q", C.c_double * (MAX_M * (MAX_M + 1))),
        ("q", C.c_double * MAX_M),
        ("Qt", C.c_double * (MAX_M * MAX_M)),
        ("S", C.c_double * (MAX_M * (MAX_M + 1))),
        ("QtI", C.c_double * (MAX_M * MAX_M)),
        ("QtE", C.c_double * (MAX_M * MAX_M)),
    ]


class CountersC(C.Structure):
    _fields_ = [
        ("diffusion", C.c_longlong),
        ("reaction", C.c_longlong),
        ("coupled", C.c_longlong),
        ("newton_iterations", C.c_longlong),
        ("mg_cycles", C.c_longlong),
    ]


class IntegrateOptionsC(C.Structure):
    _fields_ = [
        ("scheme", C.c_int),
        ("dt", C.c_double),
        ("n_steps", C.c_int),
        ("M", C.c_int),
        ("n_sweeps", C.c_int),
        ("nu", C.c_int),
        ("has_stop_tol", C.c_int),
        ("stop_tol", C.c_double),
        ("convention", C.c_int),
        ("workers", C.c_int),
    ]


class StepReportC(C.Structure):
    _fields_ = [("sweeps", C.c_int), ("counters", CountersC)]


# C-ABI symbols of include/cisdc_gpu.h: (name, restype, argtypes)
_vp = C.c_void_p
class CellTraceC(C.Structure):
    _fields_ = [("kind", C.c_int), ("m", C.c_int), ("ell", C.c_int), ("worker", C.c_int),
                ("start_ns", C.c_longlong), ("end_ns", C.c_longlong),
                ("seq_start", C.c_longlong), ("seq_end", C.c_longlong)]


class ScanPointC(C.Structure):
    """cisdc_scan_point == cisdc::ScanPoint (analysis.hpp:79-87)."""
    _fields_ = [("scheme", C.c_int), ("M", C.c_int), ("nu", C.c_int), ("a", C.c_double), ("d", C.c_double),
                ("r", C.c_double), ("dt", C.c_double), ("gamma", C.c_double), ("ok", C.c_int)]


_ip = C.POINTER(C.c_int)

GPU_SYMBOLS = [
    ("cisdc_make_quadrature_tables", C.c_int, [C.c_int, C.c_int, C.POINTER(TablesC)]),
    ("cisdc_gpu_create", C.c_int, [C.POINTER(ProblemDescC), C.POINTER(TablesC), C.POINTER(_vp)]),
    ("cisdc_gpu_destroy", None, [_vp]),
    ("cisdc_gpu_last_error", C.c_char_p, [_vp]),
    ("cisdc_gpu_dimension", C.c_size_t, [_vp]),
    ("cisdc_gpu_initialize", C.c_int, [_vp, _dp, C.c_size_t]),
    ("cisdc_gpu_initialize_device", C.c_int, [_vp, _vp, C.c_size_t]),
    ("cisdc_gpu_set_nodes", C.c_int, [_vp, _dp, C.c_size_t]),
    ("cisdc_gpu_sweep", C.c_int, [_vp, C.c_int, C.c_double, C.c_int, C.c_int, C.POINTER(CountersC)]),
    ("cisdc_gpu_increment", C.c_int, [_vp, _dp]),
    ("cisdc_gpu_get_field", C.c_int, [_vp, C.c_int, C.c_int, _dp, C.c_size_t]),
    ("cisdc_gpu_get_field_device", C.c_int, [_vp, C.c_int, C.c_int, _vp, C.c_size_t]),
    ("cisdc_gpu_eval", C.c_int, [_vp, C.c_int, _dp, _dp, C.c_size_t]),
    ("cisdc_gpu_solve", C.c_int, [_vp, C.c_int, C.c_double, _dp, _dp, C.c_size_t, C.POINTER(CountersC)]),
    ("cisdc_gpu_integrate", C.c_int,
     [_vp, _dp, C.c_size_t, C.POINTER(IntegrateOptionsC), _dp, C.POINTER(StepReportC), _dp]),
    ("cisdc_gpu_integrate_device", C.c_int,
     [_vp, _vp, C.c_size_t, C.POINTER(IntegrateOptionsC), _vp, C.POINTER(StepReportC), _dp]),
    ("cisdc_gpu_set_timing", C.c_int, [_vp, C.c_int]),
    ("cisdc_gpu_kernel_times", C.c_int, [_vp, _dp, _dp, C.POINTER(C.c_longlong), C.c_int, C.c_int]),
    ("cisdc_gpu_kernel_class_name", C.c_char_p, [C.c_int]),
    ("cisdc_gpu_device_time_ms", C.c_double, [_vp, C.c_int]),
    ("cisdc_gpu_launch_count", C.c_longlong, [_vp]),
    ("cisdc_gpu_newton_residual_exits", C.c_longlong, [_vp]),
    ("cisdc_gpu_fp64_peak", C.c_int, [_dp, _dp]),
    ("cisdc_gpu_spectral_radius_scan", C.c_int, [_ip, C.c_int, _ip, C.c_int, _dp, C.c_int, C.c_int, C.c_double,
                                                 C.c_double, C.c_double, C.c_int, C.c_int, C.POINTER(ScanPointC),
                                                 C.c_size_t, C.POINTER(C.c_size_t), _dp]),
    ("cisdc_log_r_grid", C.c_int, [C.c_double, C.c_double, C.c_int, _dp, C.c_size_t]),
    ("cisdc_gpu_spectral_radius_batch", C.c_int, [_dp, C.c_int, C.c_int, _dp, _ip]),
    ("cisdc_last_error", C.c_char_p, []),
    ("cisdc_rtc_compile_check", C.c_int, [C.POINTER(ProblemDescC), C.c_char_p, C.c_size_t]),
    ("cisdc_gpu_set_trace", C.c_int, [_vp, C.c_int]),
    ("cisdc_gpu_last_trace", C.c_int, [_vp, C.POINTER(CellTraceC), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("cisdc_write_field_snapshot", C.c_int, [C.c_char_p, C.c_int, C.c_double, _dp, C.c_size_t]),
    ("cisdc_read_field_snapshot", C.c_int, [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), _dp, C.c_size_t]),
    ("cisdc_io_last_error", C.c_char_p, []),
]

_LIB = None


def lib_path() -> str:
    from . import _build
    return _build.LIB


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load the native engine.  There is no CPU fallback: a missing library is an error."""
    global _LIB
    if _LIB is not None:
        return _LIB
    from . import _build
    if not os.path.exists(_build.LIB) or not _build.up_to_date():
        if not build_if_missing:
            raise RuntimeError(f"native engine missing: {_build.LIB}")
        _build.build()
    lib = C.CDLL(_build.LIB)
    for name, res, args in GPU_SYMBOLS:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def dptr(a) -> C.POINTER(C.c_double):
    return a.ctypes.data_as(_dp)


def iptr(a) -> C.POINTER(C.c_int):
    return a.ctypes.data_as(_ip)
