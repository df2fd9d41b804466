"""ORACLE -- TEST INFRASTRUCTURE ONLY.

ctypes access to
  * oracle/_build/libcisdc_oracle.so  -- the plain-C restatement (built from committed sources with
    gcc by ``make -C oracle``; gcc exists on the GPU box too, so tests may build it there), and
  * oracle/_ref/libcisdc_ref.so       -- the UNMODIFIED reference compiled from /root/reference
    (``make -C oracle ref``; built only where /root/reference exists, travels as a built file).
Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_1801_01201_b200 import _abi

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "_build", "libcisdc_oracle.so")
REF_LIB = os.path.join(HERE, "_ref", "libcisdc_ref.so")
ENGINE_LIB = os.path.join(HERE, "_ref", "libcisdc_engine_check.so")
REF_SRC = "/root/reference/proj/core"

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_cp = C.c_char_p
_ip = C.POINTER(C.c_int)

_oracle = None
_ref = None


def build_oracle(force: bool = False) -> str:
    srcs = [os.path.join(HERE, f) for f in ("co_numerics.c", "co_problems.c", "co_sweeps.c", "cisdc_oracle.h")]
    if force or not os.path.exists(ORACLE_LIB) or any(os.path.getmtime(s) > os.path.getmtime(ORACLE_LIB) for s in srcs):
        subprocess.run(["make", "-s", "-C", HERE, "_build/libcisdc_oracle.so"], check=True, capture_output=True)
    return ORACLE_LIB


def build_ref() -> str | None:
    if os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True, capture_output=True)
    return REF_LIB if os.path.exists(REF_LIB) else None


def build_engine_check() -> str | None:
    """integration/engine_check.cpp against the reference headers + oracle/_ref + libcisdc_gpu.so."""
    if os.path.isdir(REF_SRC):
        r = subprocess.run(["make", "-s", "-C", HERE, "engine"], capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError("engine_check build failed:\n" + r.stdout + r.stderr)
    return ENGINE_LIB if os.path.exists(ENGINE_LIB) else None


_engine = None


def engine_lib() -> C.CDLL | None:
    """The compiled reference-side consumer of the GPU engine (None when it was never built)."""
    global _engine
    if _engine is None:
        if not os.path.exists(ENGINE_LIB) and build_engine_check() is None:
            return None
        lib = C.CDLL(ENGINE_LIB)
        ll = C.POINTER(C.c_longlong)
        lib.engine_vs_reference.argtypes = [C.POINTER(_abi.ProblemDescC), _dp, C.c_size_t,
                                            C.POINTER(_abi.IntegrateOptionsC), C.c_int, _dp, _dp, ll, ll, _dp, _dp,
                                            ll, _cp, C.c_size_t]
        lib.engine_exceptions.argtypes = [C.POINTER(_abi.ProblemDescC), _dp, C.c_size_t,
                                          C.POINTER(_abi.IntegrateOptionsC), C.c_int, C.POINTER(C.c_int), _cp,
                                          C.POINTER(C.c_int), _cp, C.c_size_t]
        _engine = lib
    return _engine


def oracle_lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        build_oracle()
        lib = C.CDLL(ORACLE_LIB)
        lib.co_make_tables.argtypes = [C.c_int, C.c_int, C.POINTER(_abi.TablesC)]
        lib.co_banded_solve.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp, _cp]
        lib.co_lu_factor_dense.argtypes = [C.c_int, _dp, C.POINTER(C.c_int), C.c_int, _cp]
        lib.co_lu_solve.argtypes = [C.c_int, _dp, C.POINTER(C.c_int), _dp, _dp]
        lib.co_problem_create.argtypes = [C.POINTER(_abi.ProblemDescC), C.POINTER(_vp), _cp]
        lib.co_problem_destroy.argtypes = [_vp]
        lib.co_problem_dim.argtypes = [_vp]
        lib.co_problem_dim.restype = C.c_size_t
        lib.co_problem_error.argtypes = [_vp]
        lib.co_problem_error.restype = C.c_char_p
        lib.co_eval.argtypes = [_vp, C.c_int, _dp, _dp]
        lib.co_solve.argtypes = [_vp, C.c_int, C.c_double, _dp, _dp, C.POINTER(_abi.CountersC)]
        lib.co_state_create.argtypes = [C.c_int, C.c_size_t]
        lib.co_state_create.restype = _vp
        lib.co_state_destroy.argtypes = [_vp]
        lib.co_state_initialize.argtypes = [_vp, _vp, _dp]
        lib.co_state_set_nodes.argtypes = [_vp, _vp, _dp]
        lib.co_state_field.argtypes = [_vp, C.c_int, C.c_int]
        lib.co_state_field.restype = _dp
        lib.co_increment_norm.argtypes = [_dp, _dp, C.c_size_t]
        lib.co_increment_norm.restype = C.c_double
        lib.co_run_sweep.argtypes = [C.c_int, _vp, C.POINTER(_abi.TablesC), _vp, C.c_double, C.c_int,
                                     C.POINTER(_abi.CountersC)]
        lib.co_integrate.argtypes = [_vp, _dp, C.POINTER(_abi.IntegrateOptionsC), _dp,
                                     C.POINTER(_abi.StepReportC), _dp, _cp]
        _oracle = lib
    return _oracle


def ref_lib() -> C.CDLL | None:
    """The unmodified reference (None when it was never built here)."""
    global _ref
    if _ref is None:
        if not os.path.exists(REF_LIB):
            if build_ref() is None:
                return None
        lib = C.CDLL(REF_LIB)
        lib.ref_make_tables.argtypes = [C.c_int, C.c_int, C.POINTER(_abi.TablesC)]
        lib.ref_banded_solve.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]
        lib.ref_integrate.argtypes = [C.POINTER(_abi.ProblemDescC), _dp, C.POINTER(_abi.IntegrateOptionsC), _dp,
                                      C.POINTER(_abi.StepReportC), _dp, _cp]
        lib.ref_sweeps.argtypes = [C.POINTER(_abi.ProblemDescC), C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                   C.c_int, C.c_int, _dp, _dp, _dp, C.POINTER(_abi.CountersC), _cp]
        lib.ref_stage.argtypes = [C.POINTER(_abi.ProblemDescC), C.c_int, C.c_int, C.c_double, _dp, _dp, _cp]
        lib.ref_rd_initial_condition.argtypes = [C.c_int, C.c_double, C.c_double, C.c_double, _dp]
        lib.ref_write_field_snapshot.argtypes = [C.c_char_p, C.c_int, C.c_double, _dp, C.c_size_t, _cp]
        lib.ref_read_field_snapshot.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_double), _dp,
                                                C.c_size_t, _cp]
        lib.ref_spectral_radius.argtypes = [_dp, C.c_int, _dp]
        sp = C.POINTER(_abi.ScanPointC)
        lib.ref_spectral_radius_scan.argtypes = [_ip, C.c_int, _ip, C.c_int, _dp, C.c_int, C.c_int, C.c_double,
                                                 C.c_double, C.c_double, C.c_int, C.c_int, sp, C.c_size_t,
                                                 C.POINTER(C.c_size_t), _dp, _cp]
        tp = C.POINTER(_abi.CellTraceC)
        lib.ref_validate_trace.argtypes = [C.c_int, C.c_int, C.c_int, tp, C.c_int, _cp, C.c_size_t]
        _ref = lib
    return _ref


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _dp_of(a):
    return a.ctypes.data_as(_dp)


# ----------------------------------------------------------------------------- restatement

def make_tables(M: int, convention: int = 0) -> _abi.TablesC:
    t = _abi.TablesC()
    rc = oracle_lib().co_make_tables(M, convention, C.byref(t))
    if rc:
        raise OracleError(rc, "co_make_tables")
    return t


class Problem:
    def __init__(self, desc):
        self.desc = desc
        self._c = desc.to_c()
        self.h = _vp()
        err = C.create_string_buffer(512)
        rc = oracle_lib().co_problem_create(C.byref(self._c), C.byref(self.h), err)
        if rc:
            raise OracleError(rc, err.value.decode())
        self.n = int(oracle_lib().co_problem_dim(self.h))

    def error(self) -> str:
        return oracle_lib().co_problem_error(self.h).decode()

    def eval(self, stage: int, phi: np.ndarray) -> np.ndarray:
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        out = np.empty_like(phi)
        rc = oracle_lib().co_eval(self.h, stage, _dp_of(phi), _dp_of(out))
        if rc:
            raise OracleError(rc, self.error())
        return out

    def solve(self, stage: int, coef: float, rhs: np.ndarray, counters=None) -> np.ndarray:
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        out = np.empty_like(rhs)
        c = counters if counters is not None else _abi.CountersC()
        rc = oracle_lib().co_solve(self.h, stage, float(coef), _dp_of(rhs), _dp_of(out), C.byref(c))
        if rc:
            raise OracleError(rc, self.error())
        return out

    def __del__(self):
        if getattr(self, "h", None):
            oracle_lib().co_problem_destroy(self.h)
            self.h = None


class State:
    """co_state: the oracle's SweepState."""

    def __init__(self, problem: Problem, M: int):
        self.p = problem
        self.M = M
        self.h = oracle_lib().co_state_create(M, problem.n)

    def initialize(self, phi0):
        phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
        rc = oracle_lib().co_state_initialize(self.h, self.p.h, _dp_of(phi0))
        if rc:
            raise OracleError(rc, self.p.error())

    def set_node_values(self, values):
        v = np.ascontiguousarray(np.asarray(values, dtype=np.float64).reshape(self.M + 1, -1))
        rc = oracle_lib().co_state_set_nodes(self.h, self.p.h, _dp_of(v))
        if rc:
            raise OracleError(rc, self.p.error())

    def field(self, which: int, node: int) -> np.ndarray:
        ptr = oracle_lib().co_state_field(self.h, which, node)
        return np.ctypeslib.as_array(ptr, shape=(self.p.n,)).copy()

    def sweep(self, scheme: int, tables: _abi.TablesC, dt: float, nu: int = 1, counters=None):
        c = counters if counters is not None else _abi.CountersC()
        rc = oracle_lib().co_run_sweep(scheme, self.h, C.byref(tables), self.p.h, float(dt), int(nu), C.byref(c))
        if rc:
            raise OracleError(rc, self.p.error())

    def __del__(self):
        if getattr(self, "h", None):
            oracle_lib().co_state_destroy(self.h)
            self.h = None


def integrate(desc, phi0, opt):
    """co_integrate: returns (final_state, reports, increments) like cisdc::integrate."""
    p = Problem(desc)
    phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
    final = np.empty_like(phi0)
    reps = (_abi.StepReportC * max(opt.n_steps, 1))()
    incs = np.zeros(max(opt.n_steps * opt.n_sweeps, 1))
    err = C.create_string_buffer(1024)
    o = opt.to_c()
    rc = oracle_lib().co_integrate(p.h, _dp_of(phi0), C.byref(o), _dp_of(final), reps, _dp_of(incs), err)
    if rc:
        raise OracleError(rc, err.value.decode())
    return final, [reps[s] for s in range(opt.n_steps)], incs


def sweeps(desc, M, convention, scheme, dt, nu, n_sweeps, phi0=None, values=None):
    """Run n_sweeps on a fresh oracle state; returns fields[5, M+1, n] and counters."""
    p = Problem(desc)
    st = State(p, M)
    if values is not None:
        st.set_node_values(values)
    else:
        st.initialize(phi0)
    t = make_tables(M, convention)
    c = _abi.CountersC()
    for _ in range(n_sweeps):
        st.sweep(scheme, t, dt, nu, c)
    out = np.stack([np.stack([st.field(w, m) for m in range(M + 1)]) for w in range(5)])
    return out, c


# ----------------------------------------------------------------------------- reference

def ref_make_tables(M: int, convention: int = 0) -> _abi.TablesC:
    t = _abi.TablesC()
    rc = ref_lib().ref_make_tables(M, convention, C.byref(t))
    if rc:
        raise OracleError(rc, "ref_make_tables")
    return t


def ref_integrate(desc, phi0, opt):
    c = desc.to_c()
    phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
    final = np.empty_like(phi0)
    reps = (_abi.StepReportC * max(opt.n_steps, 1))()
    incs = np.zeros(max(opt.n_steps * opt.n_sweeps, 1))
    err = C.create_string_buffer(1024)
    o = opt.to_c()
    rc = ref_lib().ref_integrate(C.byref(c), _dp_of(phi0), C.byref(o), _dp_of(final), reps, _dp_of(incs), err)
    if rc:
        raise OracleError(rc, err.value.decode())
    return final, [reps[s] for s in range(opt.n_steps)], incs


def ref_sweeps(desc, M, convention, scheme, dt, nu, n_sweeps, phi0=None, values=None, workers=0):
    c = desc.to_c()
    n = desc.dim
    out = np.empty((5, M + 1, n))
    cnt = _abi.CountersC()
    err = C.create_string_buffer(1024)
    p0 = np.ascontiguousarray(phi0 if phi0 is not None else np.zeros(n), dtype=np.float64)
    vals = None if values is None else np.ascontiguousarray(values, dtype=np.float64).reshape(-1)
    rc = ref_lib().ref_sweeps(C.byref(c), M, convention, scheme, float(dt), nu, workers, n_sweeps, _dp_of(p0),
                              None if vals is None else _dp_of(vals), _dp_of(out), C.byref(cnt), err)
    if rc:
        raise OracleError(rc, err.value.decode())
    return out, cnt


def ref_stage(desc, solve: bool, stage: int, coef: float, x: np.ndarray) -> np.ndarray:
    c = desc.to_c()
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    err = C.create_string_buffer(1024)
    rc = ref_lib().ref_stage(C.byref(c), int(solve), stage, float(coef), _dp_of(x), _dp_of(out), err)
    if rc:
        raise OracleError(rc, err.value.decode())
    return out


# ---------------------------------------------------------------- snapshot IO / schedule traces (reference)

def ref_write_field_snapshot(path: str, n_x: int, dx: float, data) -> None:
    a = np.ascontiguousarray(data, dtype=np.float64)
    err = C.create_string_buffer(1024)
    rc = ref_lib().ref_write_field_snapshot(str(path).encode(), int(n_x), float(dx), _dp_of(a), a.size, err)
    if rc:
        raise OracleError(rc, err.value.decode())


def ref_read_field_snapshot(path: str):
    n, dx = C.c_int(), C.c_double()
    err = C.create_string_buffer(1024)
    rc = ref_lib().ref_read_field_snapshot(str(path).encode(), C.byref(n), C.byref(dx), None, 0, err)
    if rc:
        raise OracleError(rc, err.value.decode())
    out = np.empty(n.value)
    ref_lib().ref_read_field_snapshot(str(path).encode(), C.byref(n), C.byref(dx), _dp_of(out), out.size, err)
    return n.value, dx.value, out


def _trace_arrays(trace):
    buf = (_abi.CellTraceC * max(len(trace.cells), 1))()
    for i, c in enumerate(trace.cells):
        buf[i].kind, buf[i].m, buf[i].ell, buf[i].worker = int(c.cell.kind), c.cell.m, c.cell.ell, c.worker
        buf[i].start_ns, buf[i].end_ns, buf[i].seq_start, buf[i].seq_end = c.start_ns, c.end_ns, c.seq_start, c.seq_end
    return buf


def ref_validate_schedule_trace(M: int, nu: int, trace) -> str:
    """The reference's validate_schedule_trace (pipeline.cpp:322-350) on a trace in cell-id order."""
    msg = C.create_string_buffer(1024)
    rc = ref_lib().ref_validate_trace(M, nu, trace.workers, _trace_arrays(trace), len(trace.cells), msg, 1024)
    if rc:
        raise OracleError(rc, msg.value.decode())
    return msg.value.decode()


def ref_spectral_radius_scan(schemes, nu_list, r_grid, d_rule=0, fixed_d=-5.0, a=1.0, dt=1.0, M=4, convention=0,
                             want_G=False):
    """The unmodified reference's spectral_radius_scan: (points, G or None)."""
    sch = np.ascontiguousarray(schemes, dtype=np.int32)
    nus = np.ascontiguousarray(nu_list if len(nu_list) else [1], dtype=np.int32)
    rg = np.ascontiguousarray(r_grid, dtype=np.float64)
    cap = max(len(sch) * max(len(nus), 1) * max(len(rg), 1), 1)
    out = (_abi.ScanPointC * cap)()
    n = C.c_size_t()
    G = np.zeros(cap * M * M) if want_G else None
    err = C.create_string_buffer(1024)
    rc = ref_lib().ref_spectral_radius_scan(sch.ctypes.data_as(_ip), len(sch), nus.ctypes.data_as(_ip), len(nu_list),
                                            _dp_of(rg) if len(rg) else None, len(rg), d_rule, fixed_d, a, dt, M,
                                            convention, out, cap, C.byref(n), _dp_of(G) if want_G else None, err)
    if rc:
        raise OracleError(rc, err.value.decode())
    pts = [out[i] for i in range(n.value)]
    return pts, (G[: n.value * M * M].reshape(n.value, M, M) if want_G else None)


def ref_spectral_radius(A):
    """The unmodified reference's spectral_radius of one square matrix: (rho, error code)."""
    A = np.ascontiguousarray(A, dtype=np.float64)
    rho = C.c_double(0.0)
    rc = ref_lib().ref_spectral_radius(_dp_of(A), A.shape[0], C.byref(rho))
    return rho.value, rc
