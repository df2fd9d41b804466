"""IMEXQ and the linear scalar model on the GPU.

The reference has exactly one problem class with the coupled diffusion-reaction solve IMEXQ needs:
LinearScalarProblem (proj/core/include/cisdc/problems/linear.hpp:31-51, solve_coupled
linear.cpp:45-50).  The engine runs it as a batch of independent copies (n[0] elements, the same
arithmetic per element), so every test below pins the GPU against the UNMODIFIED reference
(oracle/_ref: cisdc::integrate / imexq_sweep on LinearScalarProblem, per element) and against the
restated oracle, bit for bit, and ports the reference's IMEXQ tests (test_integrators.cpp:195-235).
"""
import numpy as np
import pytest

from paper_1801_01201_b200 import _abi, api, problems as P

pytestmark = pytest.mark.gpu

MISDC, MISDCQ, CISDCQ, IMEXQ = 0, 1, 2, 3
TRIPLES = [(1.0, -2.0, -1.0), (0.5, -40.0, -3.0), (-1.0, -0.25, -1000.0)]


def opts(scheme, M, dt, steps, sweeps, nu=1, conv=0):
    return api.IntegrateOptions(scheme=scheme, dt=dt, n_steps=steps, M=M, n_sweeps=sweeps, nu=nu, convention=conv)


@pytest.mark.parametrize("tri", TRIPLES)
@pytest.mark.parametrize("scheme,nu", [(MISDC, 1), (MISDCQ, 1), (CISDCQ, 1), (CISDCQ, 3), (IMEXQ, 1)])
@pytest.mark.parametrize("conv", [0, 1])
def test_linear_scalar_vs_unmodified_reference(gpu, ref, tri, scheme, nu, conv):
    """Dimension 1 (the reference's own problem): GPU == cisdc::integrate bit for bit, per step, with the
    same sweep and stage counts (IMEXQ counts coupled solves)."""
    p = P.linear_scalar(*tri)
    o = opts(scheme, 3, 0.1, 4, 5, nu=nu, conv=conv)
    phi0 = np.array([1.0])
    g = api.integrate(p, phi0, o)
    r, reps, incs = ref.ref_integrate(p, phi0, o)
    assert np.array_equal(g.final_state, r), (g.final_state, r)
    for s, rep in zip(g.steps, reps):
        assert s.sweeps == rep.sweeps
        assert (s.counters.diffusion, s.counters.reaction, s.counters.coupled) == (
            rep.counters.diffusion, rep.counters.reaction, rep.counters.coupled)


@pytest.mark.parametrize("scheme,nu", [(MISDC, 1), (MISDCQ, 1), (CISDCQ, 2), (IMEXQ, 1)])
def test_linear_batch_vs_oracle_and_reference(gpu, oracle, scheme, nu):
    """A batch of 100 003 copies (ragged vs the block size) with seeded initial values: GPU == oracle
    (same loop per element) bitwise; sampled elements == the unmodified reference's dimension-1 run."""
    tri = (0.5, -40.0, -3.0)
    n = 100003
    rng = np.random.default_rng(11)
    phi0 = rng.uniform(-2.0, 2.0, n)
    p = P.linear_scalar(*tri, batch=n)
    o = opts(scheme, 4, 0.05, 3, 4, nu=nu)
    g = api.integrate(p, phi0, o)
    c, reps, _ = oracle.integrate(p, phi0, o)
    assert np.array_equal(g.final_state, c)
    assert g.steps[-1].counters.coupled == reps[-1].counters.coupled
    if oracle.ref_lib() is not None:
        for i in (0, 1, 77, n - 1):
            r, _, _ = oracle.ref_integrate(P.linear_scalar(*tri), phi0[i:i + 1], o)
            assert g.final_state[i] == r[0], i


def test_cisdcq_converges_to_imexq_gpu(gpu):
    """test_integrators.cpp:195-213 on the GPU sweep engine: CISDCQ with nu = 64 inner iterations
    reaches IMEXQ's sweep (1e-10) and differs from MISDCQ (> 1e-3); M = 2, cumulative convention."""
    tri = (1.0, -2.0, -1.0)
    res = {}
    for name, scheme, nu in (("c", CISDCQ, 64), ("i", IMEXQ, 1), ("m", MISDCQ, 1)):
        st = api.SweepState(P.linear_scalar(*tri), 2, api.EulerConvention.cumulative)
        st.initialize(np.array([1.0]))
        api.run_sweep(scheme, st, 1.0, nu)
        res[name] = [st.phi(m)[0] for m in (1, 2)]
        st.close()
    for k in range(2):
        assert abs(res["c"][k] - res["i"][k]) <= 1e-10
    assert abs(res["c"][1] - res["m"][1]) > 1e-3


def test_imexq_sweep_fields_and_phi_ad(gpu, oracle):
    """One IMEXQ sweep from arbitrary node values (set_node_values): every stored field (phi, F_A, F_D,
    F_R, phi_AD = phi) equals the oracle's imexq_sweep, bitwise."""
    tri = (0.3, -5.0, -7.0)
    M = 3
    rng = np.random.default_rng(3)
    vals = rng.uniform(-1, 1, (M + 1, 1))
    st = api.SweepState(P.linear_scalar(*tri), M)
    st.set_node_values(vals)
    c = api.SolveCounters()
    api.run_sweep(IMEXQ, st, 0.7, 1, counters=c)
    assert c.coupled == M and c.diffusion == 0 and c.reaction == 0
    orc = oracle.State(oracle.Problem(P.linear_scalar(*tri)), M)
    orc.set_node_values(vals)
    orc.sweep(IMEXQ, oracle.make_tables(M, 0), 0.7, 1)
    for which in (_abi.FIELD_PHI, _abi.FIELD_FA, _abi.FIELD_FD, _abi.FIELD_FR, _abi.FIELD_PHI_AD):
        for m in range(1, M + 1):
            assert np.array_equal(st.field(which, m), orc.field(which, m)), (which, m)
    st.close()


def test_coupled_stage_solve(gpu, oracle):
    """solve_coupled (linear.cpp:45-50) through the stage API == the oracle's stage solve, bitwise; the
    singular coupled stage raises the reference's SolveError."""
    tri = (0.0, -1.5, 0.5)
    prob = api.GpuProblem(P.linear_scalar(*tri, batch=5), M=2)
    orc = oracle.Problem(P.linear_scalar(*tri, batch=5))
    rhs = np.linspace(-1.0, 1.0, 5)
    assert np.array_equal(prob.solve_coupled(0.3, rhs), orc.solve(_abi.STAGE_COUPLED, 0.3, rhs))
    with pytest.raises(api.SolveError, match="LinearScalarProblem: singular coupled stage"):
        prob.solve_coupled(-1.0, rhs)  # 1 - (-1) * (-1.5 + 0.5) == 0
    prob.close()
    adr = api.GpuProblem(P.config_c1(scale=16).problem, M=2)
    with pytest.raises(api.CapabilityError):
        adr.solve_coupled(0.1, np.zeros(adr.ctx.n))
    adr.close()


def test_singular_stage_messages_match_oracle(gpu, oracle):
    """integrate where a stage factor 1 - coef * c vanishes exactly (coef = dt QtI(0,0), c = 1/coef):
    the GPU raises the oracle's error text (step / sweep prefix and the reference's message)."""
    M, dt = 2, 0.5
    t = api.make_quadrature_tables(M)
    inv = 1.0 / (dt * t.QtI[0, 0])
    cases = ((IMEXQ, (0.0, 0.5 * inv, 0.5 * inv)), (MISDCQ, (0.0, inv, -1.0)), (MISDCQ, (0.0, -1.0, inv)))
    for scheme, tri in cases:
        p = P.linear_scalar(*tri)
        o = opts(scheme, M, dt, 1, 2)
        try:
            oracle.integrate(p, np.array([1.0]), o)
            pytest.skip("stage factor did not vanish exactly in floating point")
        except oracle.OracleError as ce:
            want = str(ce).split("] ", 1)[1]
        with pytest.raises(api.SolveError) as ge:
            api.integrate(p, np.array([1.0]), o)
        assert str(ge.value) == want, (str(ge.value), want)


def test_imexq_needs_coupled_solve_gpu(gpu):
    """test_integrators.cpp:215-235: IMEXQ on a problem without a coupled solve is a CapabilityError."""
    spec = P.config_c1(scale=16)
    st = api.SweepState(spec.problem, 2)
    st.initialize(spec.phi0)
    with pytest.raises(api.CapabilityError, match="coupled"):
        api.run_sweep(IMEXQ, st, 0.1, 1)
    st.close()
