"""The reference's own known-answer tests, run against the oracle restatement (no GPU).

Ported case by case from proj/tests/test_quadrature.cpp, test_linalg.cpp and
test_integrators.cpp (file:line on each test); tolerances are the reference's.
"""
import ctypes as C
import math

import numpy as np
import pytest

from paper_1801_01201_b200 import _abi, problems as P

MISDC, MISDCQ, CISDCQ, IMEXQ = 0, 1, 2, 3


def tables(oracle, M, conv=0):
    t = oracle.make_tables(M, conv)
    a = lambda arr, r, c: np.array(arr[: r * c]).reshape(r, c)  # noqa: E731
    return t, dict(tau=np.array(t.tau[: M + 1]), dtau=np.array(t.dtau[:M]), Q=a(t.Q, M, M + 1), S=a(t.S, M, M + 1),
                   QtI=a(t.QtI, M, M), QtE=a(t.QtE, M, M), Qt=a(t.Qt, M, M), q=np.array(t.q[:M]))


# ---------------------------------------------------------------- test_quadrature.cpp

def test_nodes_endpoints_symmetry(oracle):  # test_quadrature.cpp:25-48
    for M in range(1, 9):
        _, T = tables(oracle, M)
        assert T["tau"][0] == 0.0 and T["tau"][-1] == 1.0
        assert np.all(T["dtau"] > 0)
        assert abs(T["dtau"].sum() - 1.0) <= 1e-14
        assert np.all(np.abs(T["tau"] + T["tau"][::-1] - 1.0) <= 1e-14)
    assert abs(tables(oracle, 2)[1]["tau"][1] - 0.5) <= 1e-15


def test_nodes_m4_closed_form(oracle):  # test_quadrature.cpp:50-66
    _, T = tables(oracle, 4)
    s = math.sqrt(3.0 / 7.0)
    assert abs(T["tau"][1] - 0.5 * (1 - s)) <= 1e-14
    assert abs(T["tau"][2] - 0.5) <= 1e-14
    assert abs(T["tau"][3] - 0.5 * (1 + s)) <= 1e-14
    for M in range(2, 9):
        _, T = tables(oracle, M)
        dP = np.polynomial.legendre.Legendre.basis(M).deriv()
        for j in range(1, M):
            assert abs(dP(2 * T["tau"][j] - 1)) <= 1e-11


def test_Q_exact_rows_m2(oracle):  # test_quadrature.cpp:68-78
    Q = tables(oracle, 2)[1]["Q"]
    exp = np.array([[5 / 24, 1 / 3, -1 / 24], [1 / 6, 2 / 3, 1 / 6]])
    assert np.allclose(Q, exp, rtol=1e-15, atol=0)


def test_Q_S_polynomial_exactness(oracle):  # test_quadrature.cpp:80-100
    for M in range(1, 7):
        _, T = tables(oracle, M)
        for p in range(M + 1):
            f = T["tau"] ** p
            for m in range(M):
                up, lo = T["tau"][m + 1] ** (p + 1) / (p + 1), T["tau"][m] ** (p + 1) / (p + 1)
                assert abs(T["Q"][m] @ f - up) <= 1e-13
                assert abs(T["S"][m] @ f - (up - lo)) <= 1e-13


def test_row_sums(oracle):  # test_quadrature.cpp:102-117
    """Q rows sum to tau.  The reference's 1e-14 bound FAILS at M = 6, 8 because of build_Q's own
    round-off (SURVEY.md finding 3); the restatement reproduces that round-off exactly."""
    for M in (1, 2, 3, 4, 6, 8):
        _, T = tables(oracle, M)
        for m in range(M):
            qs = sum(T["Q"][m])
            err = abs(qs - T["tau"][m + 1])
            if M <= 4:
                assert err <= 1e-14 * T["tau"][m + 1]
            else:
                assert err <= 1e-12
    # the documented failure magnitude at M = 6 (9.7e-14) is reproduced, not "fixed"
    _, T6 = tables(oracle, 6)
    worst = max(abs(sum(T6["Q"][m]) - T6["tau"][m + 1]) for m in range(6))
    assert 1e-14 < worst < 1e-12


def test_S_is_row_difference_of_Q(oracle):  # test_quadrature.cpp:119-130
    for M in (2, 4, 5):
        _, T = tables(oracle, M)
        assert np.all(np.abs(T["S"][0] - T["Q"][0]) <= 1e-15)
        assert np.all(np.abs(T["S"][1:] - (T["Q"][1:] - T["Q"][:-1])) <= 1e-15)


def test_QtI(oracle):  # test_quadrature.cpp:132-200
    _, T = tables(oracle, 2)
    assert abs(T["QtI"][0, 0] - 1 / 3) <= 1e-15 and T["QtI"][0, 1] == 0.0
    assert abs(T["QtI"][1, 0] - 2 / 3) <= 1e-15 and abs(T["QtI"][1, 1] - 0.25) <= 1e-15
    for M in range(1, 9):
        _, T = tables(oracle, M)
        assert np.all(np.diag(T["QtI"]) > 0) and np.all(np.triu(T["QtI"], 1) == 0.0)
        U, A = T["QtI"].T, T["Qt"].T
        L = A @ np.linalg.inv(U)
        assert np.allclose(np.diag(L), 1.0, atol=1e-12)
        assert np.max(np.abs(L @ U - A)) <= 1e-14


def test_QtE_conventions(oracle):  # test_quadrature.cpp:202-233
    for conv in (0, 1):
        E = tables(oracle, 2, conv)[1]["QtE"]
        assert E[0, 0] == E[0, 1] == E[1, 1] == 0.0 and abs(E[1, 0] - 0.5) <= 1e-15
    _, T = tables(oracle, 4, 0)
    assert T["QtE"][3, 2] == T["dtau"][3] and T["QtE"][3, 0] == 0.0
    _, T = tables(oracle, 4, 1)
    assert list(T["QtE"][3, :3]) == list(T["dtau"][1:4]) and T["QtE"][3, 3] == 0.0


def test_zero_pivot_reported(oracle):  # test_quadrature.cpp:192-199 (build_QtI zero pivot)
    a = np.array([0.0, 1.0, 1.0, 0.0])
    perm = (C.c_int * 2)()
    err = C.create_string_buffer(512)
    rc = oracle.oracle_lib().co_lu_factor_dense(2, a.ctypes.data_as(C.POINTER(C.c_double)), perm, 0, err)
    assert rc == _abi.E_FACTORIZATION and b"zero pivot" in err.value


# ---------------------------------------------------------------- test_linalg.cpp

def _banded(oracle, n, kl, ku, band, b):
    x = np.empty(n)
    err = C.create_string_buffer(512)
    dp = lambda v: v.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    rc = oracle.oracle_lib().co_banded_solve(n, kl, ku, dp(band), dp(b), dp(x), err)
    return rc, x, err.value


def test_banded_pentadiagonal_laplacian_vs_dense(oracle):  # test_linalg.cpp:100-122
    n, kl = 50, 2
    st = [-1.0, 16.0, -30.0, 16.0, -1.0]
    band = np.zeros(5 * n)
    A = np.zeros((n, n))
    for i in range(n):
        for o in range(-2, 3):
            j = i + o
            if 0 <= j < n:
                v = (1.0 if i == j else 0.0) - 0.05 * st[o + 2]
                band[(j - i + kl) * n + i] = v
                A[i, j] = v
    b = np.random.default_rng(11).uniform(-1, 1, n)
    rc, x, _ = _banded(oracle, n, 2, 2, band, b)
    assert rc == 0 and np.max(np.abs(x - np.linalg.solve(A, b))) <= 1e-12


def test_banded_random_vs_dense(oracle):  # test_linalg.cpp:124-146
    rng = np.random.default_rng(23)
    for n in (10, 37, 100):
        for kl in (1, 3):
            band = np.zeros((2 * kl + 1) * n)
            A = np.zeros((n, n))
            for i in range(n):
                for j in range(max(0, i - kl), min(n - 1, i + kl) + 1):
                    v = rng.uniform(-1, 1) + (4.0 if i == j else 0.0)
                    band[(j - i + kl) * n + i] = v
                    A[i, j] = v
            b = rng.uniform(-1, 1, n)
            rc, x, _ = _banded(oracle, n, kl, kl, band, b)
            assert rc == 0 and np.max(np.abs(x - np.linalg.solve(A, b))) <= 1e-11


def test_banded_singular(oracle):  # test_linalg.cpp:148-156
    band = np.zeros(9)
    band[3 + 0], band[3 + 2] = 1.0, 1.0  # diag = (1, 0, 1)
    rc, _, msg = _banded(oracle, 3, 1, 1, band, np.ones(3))
    assert rc == _abi.E_SOLVE and b"singular band" in msg


def test_newton_reaction_cell_vs_bisection(oracle):  # test_linalg.cpp:220-228 via the reference PDE cell
    """x - 0.1 r x(x-1)(x-1/2) = 0.7, r = 4: the reference problem's per-cell Newton (guess = rhs)."""
    desc = P.ProblemDesc(kind=_abi.PROBLEM_REFERENCE_RD, n=(8, 1, 1), ref_a=0.0, ref_d=0.0, ref_r=4.0)
    prob = oracle.Problem(desc)
    x = prob.solve(_abi.STAGE_REACTION, 0.1, np.full(8, 0.7))
    f = lambda v: v - 0.1 * 4 * v * (v - 1) * (v - 0.5) - 0.7  # noqa: E731
    lo, hi = 0.0, 1.0
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if f(lo) * f(mid) <= 0:
            hi = mid
        else:
            lo = mid
    assert np.all(np.abs(x - 0.5 * (lo + hi)) <= 1e-12)


# ---------------------------------------------------------------- test_integrators.cpp

def lin_state(oracle, a, d, r, M):
    p = oracle.Problem(P.linear_scalar(a, d, r))
    st = oracle.State(p, M)
    st.initialize(np.array([1.0]))
    return p, st


def phiM(st, m):
    return st.field(_abi.FIELD_PHI, m)[0]


def test_zero_coefficients_leave_state_unchanged(oracle):  # test_integrators.cpp:53-66
    t, _ = tables(oracle, 3)
    for s in (MISDC, MISDCQ, IMEXQ):
        _, st = lin_state(oracle, 0, 0, 0, 3)
        st.sweep(s, t, 1.0, 1)
        assert all(phiM(st, m) == 1.0 for m in range(4))
    for nu in (1, 2, 5):
        _, st = lin_state(oracle, 0, 0, 0, 3)
        st.sweep(CISDCQ, t, 1.0, nu)
        assert all(phiM(st, m) == 1.0 for m in range(4))


def test_node0_never_changes(oracle):  # test_integrators.cpp:68-78
    t, _ = tables(oracle, 4)
    for s in (MISDC, MISDCQ, CISDCQ, IMEXQ):
        _, st = lin_state(oracle, 1.0, -2.0, -4.0, 4)
        for _ in range(12):
            st.sweep(s, t, 1.0, 3)
            assert phiM(st, 0) == 1.0


def collocation(T, s, dt, phi0=1.0):  # oracles.cpp:68-78
    M = len(T["q"])
    A = np.eye(M) - dt * s * T["Qt"]
    return np.linalg.solve(A, phi0 * (1.0 + dt * s * T["q"]))


@pytest.mark.parametrize("triple,expected", [((1.0, 0.0, 0.0), 19.0 / 7.0), ((1.0, -2.0, -4.0), 7.0 / 67.0)])
def test_linear_fixed_points_m2(oracle, triple, expected):  # test_integrators.cpp:80-105
    for conv in (0, 1):
        t, T = tables(oracle, 2, conv)
        assert abs(collocation(T, sum(triple), 1.0)[-1] - expected) <= 1e-13 * expected
        for s in (MISDC, MISDCQ, IMEXQ):
            _, st = lin_state(oracle, *triple, 2)
            for _ in range(200):
                st.sweep(s, t, 1.0, 1)
            assert abs(phiM(st, 2) - expected) <= 1e-12 * expected
        for nu in (1, 3):
            _, st = lin_state(oracle, *triple, 2)
            for _ in range(200):
                st.sweep(CISDCQ, t, 1.0, nu)
            assert abs(phiM(st, 2) - expected) <= 1e-12 * expected


@pytest.mark.parametrize("M", [2, 4])
def test_fixed_point_equivalence(oracle, M):  # test_integrators.cpp:107-135
    triple = (1.0, -2.0, -4.0)
    t, T = tables(oracle, M, 1)
    col = collocation(T, sum(triple), 1.0)
    res = []
    for s, nu in [(MISDC, 1), (MISDCQ, 1), (IMEXQ, 1), (CISDCQ, 1), (CISDCQ, 3), (CISDCQ, 6)]:
        _, st = lin_state(oracle, *triple, M)
        for _ in range(300):
            st.sweep(s, t, 1.0, nu)
        res.append(np.array([phiM(st, m) for m in range(1, M + 1)]))
    for r in res:
        assert np.all(np.abs(r - col) <= 1e-12)
        assert np.all(np.abs(r - res[0]) <= 1e-12)


def sweeps_until(oracle, scheme, triple, M, conv, tol, cap=2000):
    t, _ = tables(oracle, M, conv)
    _, st = lin_state(oracle, *triple, M)
    prev = phiM(st, M)
    for k in range(1, cap + 1):
        st.sweep(scheme, t, 1.0, 1)
        cur = phiM(st, M)
        if abs(cur - prev) <= tol:
            return k
        prev = cur
    return cap + 1


def test_misdcq_fewer_sweeps_than_misdc(oracle):  # test_integrators.cpp:137-143
    tri = (1.0, -10.0, -20.0)
    assert sweeps_until(oracle, MISDCQ, tri, 4, 1, 1e-14) < sweeps_until(oracle, MISDC, tri, 4, 1, 1e-14)


def test_cisdcq_nu_validation(oracle):  # test_integrators.cpp:145-150
    t, _ = tables(oracle, 2)
    _, st = lin_state(oracle, 1, -1, -1, 2)
    with pytest.raises(oracle.OracleError):
        st.sweep(CISDCQ, t, 1.0, 0)


def test_incremental_reaction_form_matches_direct(oracle):  # test_integrators.cpp:152-193
    rng = np.random.default_rng(17)
    for _ in range(25):
        a, d, r = rng.uniform(-1, 1, 3)
        M = 3
        t, T = tables(oracle, M, 1)
        p = oracle.Problem(P.linear_scalar(a, d, r))
        st = oracle.State(p, M)
        vals = rng.uniform(-1, 1, M + 1)
        st.set_node_values(vals.reshape(M + 1, 1))
        fa = [a * v for v in vals]
        fd = [d * v for v in vals]
        fr = [r * v for v in vals]
        dt = 0.7
        st.sweep(CISDCQ, t, dt, 1)
        phi = [phiM(st, m) for m in range(M + 1)]
        pad = [st.field(_abi.FIELD_PHI_AD, m)[0] for m in range(M + 1)]
        for m in range(M):
            rhs = vals[0]
            for j in range(M + 1):
                rhs += dt * T["Q"][m, j] * (fa[j] + fd[j] + fr[j])
            for j in range(1, m):
                rhs += dt * T["QtE"][m, j - 1] * (a * phi[j] - fa[j])
                rhs += dt * T["QtI"][m, j - 1] * (d * phi[j] - fd[j] + r * phi[j] - fr[j])
            if m >= 1:
                rhs += dt * T["QtE"][m, m - 1] * (a * pad[m] - fa[m])
                rhs += dt * T["QtI"][m, m - 1] * (d * pad[m] - fd[m] + r * phi[m] - fr[m])
            coef = dt * T["QtI"][m, m]
            rhs += coef * (d * pad[m + 1] - fd[m + 1] + r * phi[m + 1] - fr[m + 1])
            assert abs(phi[m + 1] - rhs) <= 1e-14


def test_cisdcq_converges_to_imexq(oracle):  # test_integrators.cpp:195-213
    t, _ = tables(oracle, 2, 1)
    tri = (1.0, -2.0, -1.0)
    _, sc = lin_state(oracle, *tri, 2)
    sc.sweep(CISDCQ, t, 1.0, 64)
    _, si = lin_state(oracle, *tri, 2)
    si.sweep(IMEXQ, t, 1.0, 1)
    _, sm = lin_state(oracle, *tri, 2)
    sm.sweep(MISDCQ, t, 1.0, 1)
    for m in (1, 2):
        assert abs(phiM(sc, m) - phiM(si, m)) <= 1e-10
    assert abs(phiM(sc, 2) - phiM(sm, 2)) > 1e-3


def test_imexq_requires_coupled_solve(oracle):  # test_integrators.cpp:215-235
    spec = P.config_c1(scale=16)
    p = oracle.Problem(spec.problem)
    st = oracle.State(p, 2)
    st.initialize(spec.phi0)
    t, _ = tables(oracle, 2)
    with pytest.raises(oracle.OracleError) as e:
        st.sweep(IMEXQ, t, 0.1, 1)
    assert e.value.code == _abi.E_CAPABILITY


def test_order_per_sweep(oracle):  # test_integrators.cpp:237-269
    tri = (1.0, -1.0, -2.0)
    s = sum(tri)
    dts = [2.0 ** -e for e in range(3, 9)]

    def err(scheme, M, k, dt):
        t, _ = tables(oracle, M, 1)
        _, st = lin_state(oracle, *tri, M)
        for _ in range(k):
            st.sweep(scheme, t, dt, 1)
        return abs(phiM(st, M) - math.exp(s * dt))

    def slope(scheme, M, k):
        x = np.log(dts)
        y = np.log([err(scheme, M, k, dt) for dt in dts])
        return np.polyfit(x, y, 1)[0]

    for scheme in (MISDC, MISDCQ, CISDCQ, IMEXQ):
        for k in (1, 2, 3):
            assert abs(slope(scheme, 4, k) - (k + 1)) <= 0.3
        assert abs(slope(scheme, 1, 2) - 3.0) <= 0.3
        assert slope(scheme, 1, 3) < 3.3


def test_integrate_driver(oracle):  # test_integrators.cpp:271-333
    from paper_1801_01201_b200 import api
    lin = P.linear_scalar(0, 0, 0)
    f, reps, _ = oracle.integrate(lin, np.array([1.0]), api.IntegrateOptions(scheme=MISDCQ, dt=1.0, n_steps=1, M=2,
                                                                                n_sweeps=1))
    assert f[0] == 1.0 and len(reps) == 1
    # two converged steps = (61/37)^2
    f, reps, _ = oracle.integrate(P.linear_scalar(1, 0, 0), np.array([1.0]),
                                  api.IntegrateOptions(scheme=MISDCQ, dt=0.5, n_steps=2, M=2, n_sweeps=200,
                                                       stop_tol=1e-15))
    assert abs(f[0] - 3721.0 / 1369.0) <= 1e-12 * f[0]
    assert abs(f[0] - math.e) <= 3e-4
    # per-step reports: nu * M solves per stage per sweep
    f, reps, incs = oracle.integrate(P.linear_scalar(1, -2, -4), np.array([1.0]),
                                     api.IntegrateOptions(scheme=CISDCQ, dt=0.5, n_steps=2, M=3, n_sweeps=4, nu=2))
    for r in reps:
        assert r.sweeps == 4
        assert r.counters.diffusion == 4 * 2 * 3 and r.counters.reaction == 4 * 2 * 3
    assert np.all(incs >= 0)
    with pytest.raises(oracle.OracleError):
        oracle.integrate(P.linear_scalar(1, 0, 0), np.array([1.0]), api.IntegrateOptions(n_sweeps=0))


def test_stored_evaluations_consistent(oracle):  # test_integrators.cpp:335-348
    tri = (0.7, -1.3, -0.4)
    t, _ = tables(oracle, 3, 1)
    _, st = lin_state(oracle, *tri, 3)
    for k in range(5):
        st.sweep(MISDCQ if k % 2 == 0 else CISDCQ, t, 0.8, 2)
        for m in range(4):
            ph = phiM(st, m)
            assert abs(st.field(_abi.FIELD_FA, m)[0] - tri[0] * ph) <= 1e-13
            assert abs(st.field(_abi.FIELD_FD, m)[0] - tri[1] * ph) <= 1e-13
            assert abs(st.field(_abi.FIELD_FR, m)[0] - tri[2] * ph) <= 1e-13
