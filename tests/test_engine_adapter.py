"""The drop-in on the reference side, compiled (VERDICT r1 "make the drop-in real").

integration/cisdc/gpu.hpp (cisdc::gpu::Engine, the adapter a reference maintainer adds) is compiled
against the UNMODIFIED reference headers and library into oracle/_ref/libcisdc_engine_check.so
(integration/engine_check.cpp).  Each case runs cisdc::integrate (reference integrators.hpp:84-85)
and Engine::integrate (tables from the reference's own make_quadrature_tables) on the same inputs
inside that C++ code; the states must be bit-identical and the SweepReports equal.
"""
import ctypes as C

import numpy as np
import pytest

from paper_1801_01201_b200 import _abi, api, problems as P


@pytest.fixture(scope="module")
def eng(oracle):
    lib = oracle.engine_lib()
    if lib is None:
        pytest.skip("engine_check not built (needs /root/reference at build time)")
    return lib


def test_engine_check_library_exports(eng):
    assert hasattr(eng, "engine_vs_reference") and hasattr(eng, "engine_exceptions")


def run_both(eng, desc, phi0, o, workers=0):
    c = desc.to_c()
    oc = o.to_c()
    n = phi0.size
    phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
    g, r = np.empty(n), np.empty(n)
    gc, rc = np.zeros(4 * o.n_steps, dtype=np.int64), np.zeros(4 * o.n_steps, dtype=np.int64)
    gi, ri = np.zeros(o.n_steps * o.n_sweeps), np.zeros(o.n_steps * o.n_sweeps)
    gn = np.zeros(o.n_steps, dtype=np.int64)
    err = C.create_string_buffer(1024)
    ll = C.POINTER(C.c_longlong)
    rv = eng.engine_vs_reference(C.byref(c), _abi.dptr(phi0), n, C.byref(oc), workers, _abi.dptr(g), _abi.dptr(r),
                                 gc.ctypes.data_as(ll), rc.ctypes.data_as(ll), _abi.dptr(gi), _abi.dptr(ri),
                                 gn.ctypes.data_as(ll), err, 1024)
    assert rv == 0, err.value.decode()
    return g, r, gc, rc, gi, ri


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,nu,workers", [(0, 1, 0), (1, 1, 0), (2, 1, 0), (2, 3, 0), (2, 1, 2), (2, 3, 2)])
@pytest.mark.parametrize("conv", [0, 1])
def test_engine_equals_reference_integrate_config0(gpu, eng, scheme, nu, workers, conv):
    """The reference's own PDE (cisdc::ReactionDiffusionProblem, n_x = 200): Engine == cisdc::integrate."""
    spec = P.config_c0(n_steps=5)
    o = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=5, M=spec.M, n_sweeps=spec.n_sweeps, nu=nu,
                             convention=conv)
    g, r, gc, rc, gi, ri = run_both(eng, spec.problem, spec.phi0, o, workers)
    assert np.array_equal(g, r)
    assert np.array_equal(gc, rc)
    assert np.allclose(gi, ri, rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("scheme,workers", [(1, 0), (2, 0), (2, 2)])
def test_engine_equals_reference_integrate_scaled_c5(gpu, eng, scheme, workers):
    """Config 5 scaled to 32^3 x 9 (3-D tiled stencils, multigrid, NVRTC Newton, PMISDC streams)."""
    spec = P.config_c5(scale=8)
    o = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps, nu=1)
    g, r, gc, rc, gi, ri = run_both(eng, spec.problem, spec.phi0, o, workers)
    assert np.array_equal(g, r)
    assert np.array_equal(gc, rc)
    assert np.allclose(gi, ri, rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c2", "c5"])
def test_engine_equals_reference_imexq_adr(gpu, eng, name):
    """IMEXQ on the periodic class with its coupled stage (cisdc_gpu.h): the compiled C++ side runs the
    unmodified cisdc::integrate(Scheme::imexq) over AdrProblem::solve_coupled and Engine::integrate on
    the same descriptor; states bit-identical, reports (sweeps, coupled solves) equal."""
    import dataclasses
    spec = P.config_c2(scale=128, n_steps=1) if name == "c2" else P.config_c5(scale=16)
    prob = dataclasses.replace(spec.problem, coupled_tol=1e-13, coupled_max_iter=60)
    o = api.IntegrateOptions(scheme=3, dt=spec.dt, n_steps=1, M=3, n_sweeps=2, nu=1)
    g, r, gc, rc, gi, ri = run_both(eng, prob, spec.phi0, o, 0)
    assert np.array_equal(g, r)
    assert np.array_equal(gc, rc) and gc[3] == 6  # 3 nodes x 2 sweeps coupled solves
    assert np.allclose(gi, ri, rtol=1e-12, atol=0)


def exceptions(eng, desc, phi0, o, workers=0):
    c, oc = desc.to_c(), o.to_c()
    phi0 = np.ascontiguousarray(phi0, dtype=np.float64)
    rk, gk = C.c_int(), C.c_int()
    rw, gw = C.create_string_buffer(1024), C.create_string_buffer(1024)
    eng.engine_exceptions(C.byref(c), _abi.dptr(phi0), phi0.size, C.byref(oc), workers, C.byref(rk), rw,
                          C.byref(gk), gw, 1024)
    return rk.value, rw.value.decode(), gk.value, gw.value.decode()


@pytest.mark.gpu
def test_engine_exceptions_match_reference(gpu, eng):
    """imexq on the reference PDE: both throw SolveError("integrate: step 1, sweep 1: imexq_sweep: ...")
    (the CapabilityError wrapped by integrate, integrators.cpp:318-321); n_sweeps = 0: both
    std::invalid_argument."""
    spec = P.config_c0(n_steps=1)
    o = api.IntegrateOptions(scheme=3, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=2)
    rk, rw, gk, gw = exceptions(eng, spec.problem, spec.phi0, o)
    assert rk == gk == 2, (rk, rw, gk, gw)
    assert rw == gw, (rw, gw)
    o = api.IntegrateOptions(scheme=1, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=0)
    rk, rw, gk, gw = exceptions(eng, spec.problem, spec.phi0, o)
    assert rk == gk == 0, (rk, rw, gk, gw)
    assert rw == gw


@pytest.mark.gpu
def test_engine_newton_failure_matches_reference(gpu, eng):
    """A diverging undamped Newton (config-4 network at dt = 5e-4): both sides throw SolveError with the
    same step, sweep and first failing cell."""
    spec = P.config_c4(scale=64, n_steps=1)
    o = api.IntegrateOptions(scheme=1, dt=5e-4, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps)
    rk, rw, gk, gw = exceptions(eng, spec.problem, spec.phi0, o)
    assert rk == gk == 2, (rw, gw)
    assert rw == gw, (rw, gw)
