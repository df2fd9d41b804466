"""Host-side mirror of the reference's C++ integrator API over the native B200 engine.

Same names, argument meaning and error behaviour as proj/core/include/cisdc/*.hpp:

  Scheme, EulerConvention                     integrators.hpp:30, quadrature.hpp:42
  make_quadrature_tables(M, convention)       quadrature.cpp:147-162
  SolveCounters / SweepReport                 operator_split.hpp:57-68, sweep_state.hpp:56-60
  IntegrateOptions / IntegrateResult          integrators.hpp:64-79
  GpuProblem (OperatorSplitProblem stages)    operator_split.hpp:36-54
  SweepState (device resident)                sweep_state.hpp:33-53
  run_sweep / execute_pipelined / integrate   integrators.cpp:290-333, pipeline.cpp:171-320
  Cell / TaskGraph / build_task_graph         pipeline.hpp:26-50, pipeline.cpp:36-70
  CellTrace / ScheduleTrace                   pipeline.hpp:72-84 (GPU: per-cell stream timestamps)
  validate_schedule_trace / write_trace_csv   pipeline.cpp:322-361
  write_field_snapshot / read_field_snapshot  reaction_diffusion.cpp:230-259 ("SDC1" files)
  FactorizationError / SolveError / NumericError / CapabilityError   errors.hpp:24-45

Every call goes through the C-ABI of include/cisdc_gpu.h into libcisdc_gpu.so; nothing here
computes a field value (there is no CPU fallback).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi


class Scheme(enum.IntEnum):
    misdc = 0
    misdcq = 1
    cisdcq = 2
    imexq = 3


class EulerConvention(enum.IntEnum):
    literal = 0
    cumulative = 1


class FactorizationError(RuntimeError):
    pass


class SolveError(RuntimeError):
    pass


class NumericError(RuntimeError):
    pass


class CapabilityError(RuntimeError):
    pass


class CudaError(RuntimeError):
    pass


_ERRORS = {
    _abi.E_IO: RuntimeError,
    _abi.E_INVALID_ARGUMENT: ValueError,
    _abi.E_FACTORIZATION: FactorizationError,
    _abi.E_SOLVE: SolveError,
    _abi.E_NUMERIC: NumericError,
    _abi.E_CAPABILITY: CapabilityError,
    _abi.E_CUDA: CudaError,
}


def raise_for(code: int, msg: str) -> None:
    if code != _abi.OK:
        raise _ERRORS.get(code, RuntimeError)(msg)


@dataclass
class QuadratureTables:
    M: int
    convention: int
    tau: np.ndarray
    dtau: np.ndarray
    Q: np.ndarray
    q: np.ndarray
    Qt: np.ndarray
    S: np.ndarray
    QtI: np.ndarray
    QtE: np.ndarray
    c: _abi.TablesC = None


def tables_from_c(t: _abi.TablesC) -> QuadratureTables:
    M = t.M
    a = lambda arr, r, c: np.array(arr[: r * c]).reshape(r, c)  # noqa: E731
    return QuadratureTables(M, t.convention, np.array(t.tau[: M + 1]), np.array(t.dtau[:M]), a(t.Q, M, M + 1),
                            np.array(t.q[:M]), a(t.Qt, M, M), a(t.S, M, M + 1), a(t.QtI, M, M), a(t.QtE, M, M), t)


def make_quadrature_tables(M: int, convention: int = EulerConvention.literal) -> QuadratureTables:
    lib = _abi.load()
    t = _abi.TablesC()
    rc = lib.cisdc_make_quadrature_tables(int(M), int(convention), C.byref(t))
    if rc == _abi.E_INVALID_ARGUMENT:
        raise ValueError("gauss_lobatto_nodes: M must be >= 1 (and <= 8)")
    raise_for(rc, "make_quadrature_tables failed")
    return tables_from_c(t)


@dataclass
class SolveCounters:
    diffusion: int = 0
    reaction: int = 0
    coupled: int = 0
    newton_iterations: int = 0
    mg_cycles: int = 0

    @staticmethod
    def from_c(c: _abi.CountersC) -> "SolveCounters":
        return SolveCounters(c.diffusion, c.reaction, c.coupled, c.newton_iterations, c.mg_cycles)

    def add_c(self, c: _abi.CountersC) -> None:
        self.diffusion += c.diffusion
        self.reaction += c.reaction
        self.coupled += c.coupled
        self.newton_iterations += c.newton_iterations
        self.mg_cycles += c.mg_cycles


@dataclass
class SweepReport:
    increments: list = field(default_factory=list)
    sweeps: int = 0
    counters: SolveCounters = field(default_factory=SolveCounters)


@dataclass
class IntegrateOptions:
    scheme: int = Scheme.misdcq
    dt: float = 0.0
    n_steps: int = 1
    M: int = 4
    n_sweeps: int = 1
    nu: int = 1
    stop_tol: Optional[float] = None
    convention: int = EulerConvention.literal
    workers: int = 0  # CISDCQ: 0 = serial cell order, > 0 = concurrent D/R streams (execute_pipelined)

    def to_c(self) -> _abi.IntegrateOptionsC:
        o = _abi.IntegrateOptionsC()
        o.scheme, o.dt, o.n_steps, o.M = int(self.scheme), float(self.dt), int(self.n_steps), int(self.M)
        o.n_sweeps, o.nu = int(self.n_sweeps), int(self.nu)
        o.has_stop_tol = 0 if self.stop_tol is None else 1
        o.stop_tol = 0.0 if self.stop_tol is None else float(self.stop_tol)
        o.convention, o.workers = int(self.convention), int(self.workers)
        return o


@dataclass
class IntegrateResult:
    final_state: np.ndarray
    steps: list


class GpuContext:
    """One device-resident sweep state + problem (cisdc_gpu_ctx)."""

    def __init__(self, problem, M: int, convention: int = EulerConvention.literal):
        self.lib = _abi.load()
        self.problem = problem
        self.tables = make_quadrature_tables(M, convention)
        self._desc = problem.to_c()
        h = C.c_void_p()
        rc = self.lib.cisdc_gpu_create(C.byref(self._desc), C.byref(self.tables.c), C.byref(h))
        self.h = h
        if rc != _abi.OK:
            msg = self.last_error()
            self.close()
            raise_for(rc, msg)
        self.n = int(self.lib.cisdc_gpu_dimension(self.h))
        self.M = M

    def last_error(self) -> str:
        if not self.h:
            return "no context"
        return self.lib.cisdc_gpu_last_error(self.h).decode()

    def check(self, rc: int) -> None:
        if rc != _abi.OK:
            raise_for(rc, self.last_error())

    def close(self) -> None:
        if getattr(self, "h", None):
            self.lib.cisdc_gpu_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


class GpuProblem:
    """OperatorSplitProblem stages (eval_*/solve_*) on the GPU; host arrays in and out."""

    def __init__(self, desc, M: int = 4):
        self.desc = desc
        self.ctx = GpuContext(desc, M)

    def dimension(self) -> int:
        return self.ctx.n

    def _eval(self, stage: int, phi: np.ndarray) -> np.ndarray:
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        out = np.empty_like(phi)
        self.ctx.check(self.ctx.lib.cisdc_gpu_eval(self.ctx.h, stage, _abi.dptr(phi), _abi.dptr(out), phi.size))
        return out

    def eval_advection(self, phi):
        return self._eval(_abi.STAGE_ADVECTION, phi)

    def eval_diffusion(self, phi):
        return self._eval(_abi.STAGE_DIFFUSION, phi)

    def eval_reaction(self, phi):
        return self._eval(_abi.STAGE_REACTION, phi)

    def _solve(self, stage: int, coef: float, rhs: np.ndarray, counters: Optional[SolveCounters]):
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.empty_like(rhs)
        c = _abi.CountersC()
        self.ctx.check(self.ctx.lib.cisdc_gpu_solve(self.ctx.h, stage, float(coef), _abi.dptr(rhs), _abi.dptr(out),
                                                    rhs.size, C.byref(c)))
        if counters is not None:
            counters.add_c(c)
        return out

    def solve_diffusion(self, coef, rhs, counters=None):
        return self._solve(_abi.STAGE_DIFFUSION, coef, rhs, counters)

    def solve_reaction(self, coef, rhs, counters=None):
        return self._solve(_abi.STAGE_REACTION, coef, rhs, counters)

    def solve_coupled(self, coef, rhs, counters=None):
        """phi - coef (F_D + F_R)(phi) = rhs (operator_split.hpp:49-50); problems without a coupled solve
        raise CapabilityError, as in the reference."""
        return self._solve(_abi.STAGE_COUPLED, coef, rhs, counters)

    def close(self):
        self.ctx.close()


class SweepState:
    """Device-resident SweepState (sweep_state.hpp:33-53) bound to one problem and node set."""

    def __init__(self, problem_desc, M: int, convention: int = EulerConvention.literal):
        self.ctx = GpuContext(problem_desc, M, convention)
        self.M = M

    def subintervals(self) -> int:
        return self.M

    def dim(self) -> int:
        return self.ctx.n

    def initialize(self, phi0: np.ndarray) -> None:
        phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
        self.ctx.check(self.ctx.lib.cisdc_gpu_initialize(self.ctx.h, _abi.dptr(phi0), phi0.size))

    def set_node_values(self, values) -> None:
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(self.M + 1, -1))
        self.ctx.check(self.ctx.lib.cisdc_gpu_set_nodes(self.ctx.h, _abi.dptr(v), v.shape[1]))

    def field(self, which: int, node: int) -> np.ndarray:
        out = np.empty(self.ctx.n)
        self.ctx.check(self.ctx.lib.cisdc_gpu_get_field(self.ctx.h, which, node, _abi.dptr(out), out.size))
        return out

    def phi(self, m):
        return self.field(_abi.FIELD_PHI, m)

    def fa(self, m):
        return self.field(_abi.FIELD_FA, m)

    def fd(self, m):
        return self.field(_abi.FIELD_FD, m)

    def fr(self, m):
        return self.field(_abi.FIELD_FR, m)

    def phi_ad(self, m):
        return self.field(_abi.FIELD_PHI_AD, m)

    def increment(self) -> float:
        v = C.c_double()
        self.ctx.check(self.ctx.lib.cisdc_gpu_increment(self.ctx.h, C.byref(v)))
        return v.value

    def close(self):
        self.ctx.close()


def run_sweep(scheme: int, state: SweepState, dt: float, nu: int = 1, counters: Optional[SolveCounters] = None,
              workers: int = 0) -> None:
    c = _abi.CountersC()
    state.ctx.check(state.ctx.lib.cisdc_gpu_sweep(state.ctx.h, int(scheme), float(dt), int(nu), int(workers),
                                                  C.byref(c)))
    if counters is not None:
        counters.add_c(c)


class CellKind(enum.IntEnum):
    diffusion = 0
    reaction = 1


@dataclass(frozen=True)
class Cell:
    kind: CellKind
    m: int
    ell: int


def cell_label(c: Cell) -> str:
    """pipeline.cpp cell_label: D(m,ell) / R(m,ell)."""
    return f"{'D' if c.kind == CellKind.diffusion else 'R'}({c.m},{c.ell})"


@dataclass
class TaskGraph:
    M: int
    nu: int
    cells: list
    dependencies: list
    dependents: list

    def cell_id(self, kind: int, m: int, ell: int) -> int:
        return 2 * ((ell - 1) * self.M + (m - 1)) + (1 if kind == CellKind.reaction else 0)


def build_task_graph(M: int, nu: int) -> TaskGraph:
    """The CISDCQ-nu cell DAG (pipeline.cpp:36-70):
    D(m,l) <- D(m-1,l), R(m-2,l), R(m-1,l-1), R(m,l-1);  R(m,l) <- D(m,l), R(m-1,l)."""
    if M < 1 or nu < 1:
        raise ValueError("build_task_graph: M and nu must be >= 1")
    g = TaskGraph(M, nu, [], [], [])
    for ell in range(1, nu + 1):
        for m in range(1, M + 1):
            g.cells += [Cell(CellKind.diffusion, m, ell), Cell(CellKind.reaction, m, ell)]
    g.dependencies = [[] for _ in g.cells]
    g.dependents = [[] for _ in g.cells]

    def edge(u, v):
        g.dependencies[v].append(u)
        g.dependents[u].append(v)

    for ell in range(1, nu + 1):
        for m in range(1, M + 1):
            d, r = g.cell_id(CellKind.diffusion, m, ell), g.cell_id(CellKind.reaction, m, ell)
            if m >= 2:
                edge(g.cell_id(CellKind.diffusion, m - 1, ell), d)
            if m >= 3:
                edge(g.cell_id(CellKind.reaction, m - 2, ell), d)
            if ell >= 2:
                if m >= 2:
                    edge(g.cell_id(CellKind.reaction, m - 1, ell - 1), d)
                edge(g.cell_id(CellKind.reaction, m, ell - 1), d)
            edge(d, r)
            if m >= 2:
                edge(g.cell_id(CellKind.reaction, m - 1, ell), r)
    return g


@dataclass
class CellTrace:
    cell: Cell
    worker: int
    start_ns: int
    end_ns: int
    seq_start: int
    seq_end: int


@dataclass
class ScheduleTrace:
    """pipeline.hpp:81-84.  On the GPU a worker is a stream (0: diffusion, 1: reaction) and the
    times are GPU event timestamps from the sweep's first cell."""
    workers: int
    cells: list


def validate_schedule_trace(graph: TaskGraph, trace: ScheduleTrace) -> str:
    """pipeline.cpp:322-350: '' if every DAG edge is respected in time and in the global order and
    no worker runs two cells at once, else the first violation."""
    n = len(graph.cells)
    if len(trace.cells) != n:
        return "trace size does not match graph"
    for v in range(n):
        for u in graph.dependencies[v]:
            if trace.cells[u].end_ns > trace.cells[v].start_ns or trace.cells[u].seq_end > trace.cells[v].seq_start:
                return f"edge violated: {cell_label(graph.cells[u])} -> {cell_label(graph.cells[v])}"
    by_worker = [[] for _ in range(trace.workers)]
    for c in trace.cells:
        if c.worker < 0 or c.worker >= trace.workers:
            return "bad worker id in trace"
        by_worker[c.worker].append(c)
    for w in by_worker:
        w.sort(key=lambda c: c.start_ns)
        for a, b in zip(w, w[1:]):
            if b.start_ns < a.end_ns:
                return f"worker overlap: {cell_label(a.cell)} and {cell_label(b.cell)}"
    return ""


def write_trace_csv(path: str, trace: ScheduleTrace) -> None:
    """pipeline.cpp:352-361 schema: cell,kind,m,ell,worker,start_ns,end_ns."""
    try:
        f = open(path, "w")
    except OSError:
        raise RuntimeError("write_trace_csv: cannot open " + path) from None
    with f:
        f.write("cell,kind,m,ell,worker,start_ns,end_ns\n")
        for c in trace.cells:
            f.write(f"{cell_label(c.cell)},{'D' if c.cell.kind == CellKind.diffusion else 'R'},{c.cell.m},"
                    f"{c.cell.ell},{c.worker},{c.start_ns},{c.end_ns}\n")


def last_schedule_trace(ctx: "GpuContext") -> ScheduleTrace:
    n, w = C.c_int(), C.c_int()
    ctx.check(ctx.lib.cisdc_gpu_last_trace(ctx.h, None, 0, C.byref(n), C.byref(w)))
    buf = (_abi.CellTraceC * max(n.value, 1))()
    ctx.check(ctx.lib.cisdc_gpu_last_trace(ctx.h, buf, n.value, C.byref(n), C.byref(w)))
    cells = [CellTrace(Cell(CellKind(c.kind), c.m, c.ell), c.worker, c.start_ns, c.end_ns, c.seq_start, c.seq_end)
             for c in buf[: n.value]]
    return ScheduleTrace(w.value, cells)


def execute_pipelined(state: SweepState, dt: float, nu: int, workers: int = 2,
                      counters: Optional[SolveCounters] = None) -> ScheduleTrace:
    """pipeline.cpp:171-320: one CISDCQ-nu sweep as the cell DAG (here: two CUDA streams with event
    edges), bitwise equal to cisdcq_sweep; returns the schedule trace of the run."""
    if workers < 1:
        raise ValueError("execute_pipelined: workers must be >= 1")
    state.ctx.check(state.ctx.lib.cisdc_gpu_set_trace(state.ctx.h, 1))
    try:
        run_sweep(Scheme.cisdcq, state, dt, nu, counters, workers)
        return last_schedule_trace(state.ctx)
    finally:
        state.ctx.lib.cisdc_gpu_set_trace(state.ctx.h, 0)


@dataclass
class FieldSnapshot:
    n_x: int
    dx: float
    data: np.ndarray


def write_field_snapshot(path: str, n_x: int, dx: float, data) -> None:
    """reaction_diffusion.cpp:230-244 ("SDC1", u32 n_x, f64 dx, n_x doubles)."""
    lib = _abi.load()
    a = np.ascontiguousarray(data, dtype=np.float64)
    rc = lib.cisdc_write_field_snapshot(str(path).encode(), int(n_x), float(dx), _abi.dptr(a), a.size)
    raise_for(rc, lib.cisdc_io_last_error().decode())


def read_field_snapshot(path: str) -> FieldSnapshot:
    """reaction_diffusion.cpp:246-259."""
    lib = _abi.load()
    n, dx = C.c_int(), C.c_double()
    rc = lib.cisdc_read_field_snapshot(str(path).encode(), C.byref(n), C.byref(dx), None, 0)
    raise_for(rc, lib.cisdc_io_last_error().decode())
    out = np.empty(n.value)
    rc = lib.cisdc_read_field_snapshot(str(path).encode(), C.byref(n), C.byref(dx), _abi.dptr(out), out.size)
    raise_for(rc, lib.cisdc_io_last_error().decode())
    return FieldSnapshot(n.value, dx.value, out)


def integrate(problem_desc, phi0: np.ndarray, opt: IntegrateOptions, ctx: Optional[GpuContext] = None) -> IntegrateResult:
    """cisdc::integrate (integrators.cpp:301-333) through cisdc_gpu_integrate."""
    if opt.n_sweeps < 1:
        raise ValueError("integrate: n_sweeps must be >= 1")
    if opt.scheme == Scheme.cisdcq and opt.nu < 1:
        raise ValueError("integrate: nu must be >= 1")
    own = ctx is None
    if own:
        ctx = GpuContext(problem_desc, opt.M, opt.convention)
    try:
        phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
        final = np.empty_like(phi0)
        reps = (_abi.StepReportC * max(opt.n_steps, 1))()
        incs = np.zeros(max(opt.n_steps * opt.n_sweeps, 1))
        o = opt.to_c()
        ctx.check(ctx.lib.cisdc_gpu_integrate(ctx.h, _abi.dptr(phi0), phi0.size, C.byref(o), _abi.dptr(final), reps,
                                              _abi.dptr(incs)))
        steps = []
        for s in range(opt.n_steps):
            r = reps[s]
            steps.append(SweepReport(list(incs[s * opt.n_sweeps: s * opt.n_sweeps + r.sweeps]), r.sweeps,
                                     SolveCounters.from_c(r.counters)))
        return IntegrateResult(final, steps)
    finally:
        if own:
            ctx.close()


# ----------------------------------------------------------------------------- iteration-matrix scans

@dataclass
class ScanOptions:
    """cisdc::ScanOptions (analysis.hpp:63-76)."""
    schemes: list
    nu_list: list = None
    r_grid: list = None
    d_rule: int = 0          # DRule::half_of_r (d = r / 2); 1 = fixed
    fixed_d: float = -5.0
    a: float = 1.0
    dt: float = 1.0
    M: int = 4
    convention: int = EulerConvention.literal


@dataclass
class ScanPoint:
    scheme: int
    M: int
    nu: int
    a: float
    d: float
    r: float
    dt: float
    gamma: float
    ok: bool


def log_r_grid(lo_exp: float = -2.0, hi_exp: float = 6.0, points_per_decade: int = 40) -> np.ndarray:
    """cisdc::log_r_grid (analysis.cpp:255-266), evaluated by the library (same std::pow)."""
    lib = _abi.load()
    n = lib.cisdc_log_r_grid(lo_exp, hi_exp, points_per_decade, None, 0)
    if n < 0:
        raise ValueError(lib.cisdc_last_error().decode())
    out = np.empty(n)
    lib.cisdc_log_r_grid(lo_exp, hi_exp, points_per_decade, _abi.dptr(out), n)
    return out


def spectral_radius_scan(opt: ScanOptions, return_matrices: bool = False):
    """cisdc::spectral_radius_scan (analysis.cpp:270-293) on the GPU: one thread per (scheme, nu, r)
    point builds the affine iteration matrix of one sweep on the linear model and its spectral
    radius.  Returns the points (and the M x M matrices G when asked)."""
    lib = _abi.load()
    sch = np.ascontiguousarray(opt.schemes, dtype=np.int32)
    nus = np.ascontiguousarray(opt.nu_list or [], dtype=np.int32)
    rg = np.ascontiguousarray(opt.r_grid if opt.r_grid is not None else [], dtype=np.float64)
    groups = sum(len(nus) if s == Scheme.cisdcq else 1 for s in sch)
    cap = max(groups * len(rg), 1)
    out = (_abi.ScanPointC * cap)()
    n = C.c_size_t()
    G = np.zeros(cap * opt.M * opt.M) if return_matrices else None
    ip = C.POINTER(C.c_int)
    rc = lib.cisdc_gpu_spectral_radius_scan(sch.ctypes.data_as(ip), len(sch),
                                            nus.ctypes.data_as(ip) if len(nus) else None, len(nus),
                                            _abi.dptr(rg) if len(rg) else None, len(rg), int(opt.d_rule),
                                            float(opt.fixed_d), float(opt.a), float(opt.dt), int(opt.M),
                                            int(opt.convention), out, cap, C.byref(n),
                                            _abi.dptr(G) if return_matrices else None)
    raise_for(rc, lib.cisdc_last_error().decode())
    pts = [ScanPoint(p.scheme, p.M, p.nu, p.a, p.d, p.r, p.dt, p.gamma, bool(p.ok)) for p in out[: n.value]]
    if return_matrices:
        return pts, G[: n.value * opt.M * opt.M].reshape(n.value, opt.M, opt.M)
    return pts


def spectral_radius_batch(A: np.ndarray):
    """cisdc::spectral_radius (linalg.cpp:197-332) of a batch of n x n matrices (n <= 8), one GPU thread
    each.  Returns (rho, status): status 0 ok, 1 non-finite entry, 2 QR iteration cap."""
    lib = _abi.load()
    A = np.ascontiguousarray(A, dtype=np.float64)
    if A.ndim == 2:
        A = A[None]
    count, n = A.shape[0], A.shape[1]
    rho = np.zeros(count)
    st = np.zeros(count, dtype=np.int32)
    rc = lib.cisdc_gpu_spectral_radius_batch(_abi.dptr(A), n, count, _abi.dptr(rho), st.ctypes.data_as(C.POINTER(C.c_int)))
    raise_for(rc, lib.cisdc_last_error().decode())
    return rho, st
