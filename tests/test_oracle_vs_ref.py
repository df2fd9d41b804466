"""Pin the C restatement (oracle/) against the UNMODIFIED reference compiled from /root/reference.

Bit-for-bit: quadrature tables, banded_solve, and whole integrate() runs of every scheme on the
reference's own Dirichlet PDE; and the reference's integrators driving the oracle's periodic problem
class (configs 1-5) against the oracle's restated integrators, serial and pipelined.
"""
import numpy as np
import pytest

from paper_1801_01201_b200 import api, problems as P


@pytest.mark.parametrize("M", range(1, 9))
@pytest.mark.parametrize("conv", [0, 1])
def test_tables_bitwise(ref, M, conv):
    assert bytes(ref.make_tables(M, conv)) == bytes(ref.ref_make_tables(M, conv))


def test_product_tables_bitwise(ref):
    """The product's host tables (csrc/quadrature.cpp) equal the reference's."""
    for M in range(1, 9):
        for conv in (0, 1):
            t = api.make_quadrature_tables(M, conv).c
            assert bytes(t) == bytes(ref.ref_make_tables(M, conv)), (M, conv)


def _band(n, kl, ku, rng, diag=4.0):
    band = np.zeros((kl + ku + 1) * n)
    for i in range(n):
        for j in range(max(0, i - kl), min(n - 1, i + ku) + 1):
            band[(j - i + kl) * n + i] = rng.uniform(-1, 1) + (diag if i == j else 0.0)
    return band


@pytest.mark.parametrize("n,kl", [(10, 1), (37, 3), (100, 3), (64, 4)])
def test_banded_solve_bitwise(ref, n, kl):
    import ctypes as C
    rng = np.random.default_rng(23 + n)
    band = _band(n, kl, kl, rng)
    b = rng.uniform(-1, 1, n)
    x1, x2 = np.empty(n), np.empty(n)
    err = C.create_string_buffer(512)
    dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    assert ref.oracle_lib().co_banded_solve(n, kl, kl, dp(band), dp(b), dp(x1), err) == 0
    assert ref.ref_lib().ref_banded_solve(n, kl, kl, dp(band), dp(b), dp(x2)) == 0
    assert np.array_equal(x1, x2)


@pytest.mark.parametrize("scheme,nu", [(0, 1), (1, 1), (2, 1), (2, 3)])
@pytest.mark.parametrize("conv", [0, 1])
def test_reference_pde_integrate_bitwise(ref, scheme, nu, conv):
    spec = P.config_c0(n_x=64, n_steps=3)
    opt = api.IntegrateOptions(scheme=scheme, dt=0.05, n_steps=3, M=4, n_sweeps=4, nu=nu, convention=conv)
    f1, r1, i1 = ref.integrate(spec.problem, spec.phi0, opt)
    f2, r2, i2 = ref.ref_integrate(spec.problem, spec.phi0, opt)
    assert np.array_equal(f1, f2)
    assert np.array_equal(i1, i2)
    for a, b in zip(r1, r2):
        assert a.sweeps == b.sweeps
        assert (a.counters.diffusion, a.counters.reaction) == (b.counters.diffusion, b.counters.reaction)


def _small(name):
    return {"c1": lambda: P.config_c1(scale=4), "c2": lambda: P.config_c2(scale=256, n_steps=3),
            "c3": lambda: P.config_c3(scale=32, n_steps=1), "c4": lambda: P.config_c4(scale=64, n_steps=1),
            "c5": lambda: P.config_c5(scale=16)}[name]()


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
@pytest.mark.parametrize("scheme", [0, 1, 2])
def test_periodic_problem_driven_by_reference_integrators(ref, name, scheme):
    """Reference integrate() + the oracle's periodic ADR problem == the oracle's own integrate()."""
    spec = _small(name)
    steps = min(spec.n_steps, 2)
    opt = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=steps, M=spec.M, n_sweeps=spec.n_sweeps, nu=1)
    f1, r1, i1 = ref.integrate(spec.problem, spec.phi0, opt)
    f2, r2, i2 = ref.ref_integrate(spec.problem, spec.phi0, opt)
    assert np.array_equal(f1, f2)
    assert np.array_equal(i1, i2)
    assert sum(r.counters.newton_iterations for r in r1) == r2[0].counters.newton_iterations


@pytest.mark.parametrize("nu,workers", [(1, 2), (3, 4)])
def test_pipelined_reference_equals_serial_oracle(ref, nu, workers):
    """execute_pipelined (threads) of the reference is bitwise the oracle's serial cisdcq order."""
    spec = P.config_c2(scale=256, n_steps=2)
    opt = api.IntegrateOptions(scheme=2, dt=spec.dt, n_steps=2, M=spec.M, n_sweeps=3, nu=nu, workers=workers)
    f1, _, _ = ref.integrate(spec.problem, spec.phi0, opt)
    f2, _, _ = ref.ref_integrate(spec.problem, spec.phi0, opt)
    assert np.array_equal(f1, f2)


def test_reference_initial_condition_matches_config0(ref):
    import ctypes as C
    spec = P.config_c0()
    out = np.empty(200)
    ref.ref_lib().ref_rd_initial_condition(200, 1.0, 2.0, 4.0, out.ctypes.data_as(C.POINTER(C.c_double)))
    assert np.array_equal(out, spec.phi0)


@pytest.mark.parametrize("scheme", [0, 1, 2, 3])
def test_linear_batch_oracle_vs_reference_per_element(ref, scheme):
    """The oracle's batched LinearScalarProblem (n[0] independent copies, the GPU engine's layout) equals
    the unmodified reference's dimension-1 integrate element by element; scheme 3 is IMEXQ with the
    coupled solve (integrators.cpp:145-173, linear.cpp:45-50)."""
    from paper_1801_01201_b200 import api, problems as P
    tri = (0.5, -40.0, -3.0)
    phi0 = np.linspace(-1.5, 2.0, 7)
    o = api.IntegrateOptions(scheme=scheme, dt=0.05, n_steps=2, M=3, n_sweeps=4, nu=2)
    c, reps, _ = ref.integrate(P.linear_scalar(*tri, batch=phi0.size), phi0, o)
    for i in range(phi0.size):
        r, rreps, _ = ref.ref_integrate(P.linear_scalar(*tri), phi0[i:i + 1], o)
        assert c[i] == r[0]
        assert reps[-1].counters.coupled == rreps[-1].counters.coupled
