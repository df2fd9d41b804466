"""B200-native MISDC / MISDCQ / CISDCQ ("PMISDC") sweep engine for advection-diffusion-reaction.

Drop-in for the per-sweep hot path of the reference's C++ integrators (arXiv:1801.01201,
``cisdc``): the C-ABI is include/cisdc_gpu.h, the native library is built in-tree from csrc/
(``python -m paper_1801_01201_b200._build``), and ``api`` mirrors the reference's integrator API.
"""
from . import _abi, problems  # noqa: F401
from .api import (CapabilityError, CudaError, EulerConvention, FactorizationError, GpuContext,  # noqa: F401
                  GpuProblem, IntegrateOptions, IntegrateResult, NumericError, Scheme, SolveCounters, SolveError,
                  SweepReport, SweepState, execute_pipelined, integrate, make_quadrature_tables, run_sweep)

__all__ = [
    "Scheme", "EulerConvention", "IntegrateOptions", "IntegrateResult", "SolveCounters", "SweepReport",
    "SweepState", "GpuProblem", "GpuContext", "run_sweep", "execute_pipelined", "integrate",
    "make_quadrature_tables", "FactorizationError", "SolveError", "NumericError", "CapabilityError", "CudaError",
    "problems",
]
