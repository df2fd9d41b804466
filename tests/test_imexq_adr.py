"""IMEXQ on the periodic ADR class: the coupled diffusion-reaction stage.

The reference's imexq_sweep (proj/core/src/integrators.cpp:145-173) needs the problem's
solve_coupled (operator_split.hpp:49-53); its own PDE class has none.  The periodic ADR class
defines one (include/cisdc_gpu.h, "coupled stage"): the fixed point of the alternating diffusion /
reaction stage solves -- the nested iteration of cisdcq_cells at one node (integrators.cpp:195-258),
whose limit is the coupled solve (test_integrators.cpp:195-213) -- run to convergence.

CPU tests: the restated oracle against the fixture written by the UNMODIFIED reference's imexq_sweep
driving that stage (tests/golden/imexq_adr.npz, make_golden.py --imexq) and, where oracle/_ref is
built, against the reference directly.  GPU tests (-m gpu): the engine against the oracle and the
fixture, bit for bit, through the C-ABI.
"""
import dataclasses
import os
import sys

import numpy as np
import pytest

from paper_1801_01201_b200 import _abi, api, problems as P

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402

MISDCQ, CISDCQ, IMEXQ = 1, 2, 3


def fixture():
    return np.load(os.path.join(HERE, "imexq_adr.npz"))


def with_coupled(problem, tol=1e-13, max_iter=60):
    return dataclasses.replace(problem, coupled_tol=tol, coupled_max_iter=max_iter)


def totals(reps):
    """(sweeps per step, coupled solves per step, Newton trips, multigrid cycles) of a run."""
    return ([r.sweeps for r in reps], [r.counters.coupled for r in reps],
            sum(max(r.counters.newton_iterations, 0) for r in reps), sum(max(r.counters.mg_cycles, 0) for r in reps))


def check_against_fixture(name, final, sweeps, coupled, newton, mg):
    g = fixture()
    assert np.array_equal(final, g[f"{name}_final"]), name
    c = g[f"{name}_counts"]
    assert list(sweeps) == list(c[:, 0]) and list(coupled) == list(c[:, 1]), name
    # the reference adapter reports the whole run's Newton / multigrid work on step 0
    assert newton == c[0, 2] and mg == c[0, 3], (name, newton, mg, c.tolist())


# ------------------------------------------------------------------ CPU: oracle


@pytest.mark.parametrize("name", list(MG.IMEXQ_ADR))
def test_oracle_imexq_adr_matches_reference_fixture(oracle, name):
    spec, prob, o = MG.imexq_adr_case(name)
    assert np.array_equal(spec.phi0, fixture()[f"{name}_phi0"])
    f, reps, incs = oracle.integrate(prob, spec.phi0, o)
    check_against_fixture(name, f, *totals(reps))
    assert np.array_equal(incs, fixture()[f"{name}_incs"])


@pytest.mark.parametrize("name", ["c1", "c3"])
def test_oracle_imexq_adr_vs_unmodified_reference(oracle, ref, name):
    """Where oracle/_ref is built: the unmodified imexq_sweep driving AdrProblem::solve_coupled, other
    parameters than the fixture's (M = 4, cumulative convention)."""
    spec, prob, _ = MG.imexq_adr_case(name)
    o = api.IntegrateOptions(scheme=IMEXQ, dt=spec.dt, n_steps=1, M=4, n_sweeps=2, nu=1, convention=1)
    f, reps, incs = oracle.integrate(prob, spec.phi0, o)
    r, rreps, rincs = ref.ref_integrate(prob, spec.phi0, o)
    assert np.array_equal(f, r)
    assert np.array_equal(incs, rincs)
    assert [x.counters.coupled for x in reps] == [x.counters.coupled for x in rreps]


def test_oracle_coupled_stage_solves_the_coupled_equation(oracle):
    """phi - coef (F_D(phi) + F_R(phi)) = rhs to the iteration tolerance, on a 2-D multigrid problem."""
    spec, prob, _ = MG.imexq_adr_case("c3")
    orc = oracle.Problem(prob)
    coef = 0.4 * spec.dt
    rhs = spec.phi0
    phi = orc.solve(_abi.STAGE_COUPLED, coef, rhs)
    res = phi - coef * (orc.eval(_abi.STAGE_DIFFUSION, phi) + orc.eval(_abi.STAGE_REACTION, phi)) - rhs
    assert np.abs(res).max() <= 1e-9 * np.abs(rhs).max()
    assert np.abs(phi - rhs).max() > 0.0


def test_oracle_cisdcq_inner_iterations_reach_imexq_adr(oracle):
    """test_integrators.cpp:195-213 on the PDE class: CISDCQ's nested iteration converges to the IMEXQ
    sweep (the coupled solve), not to MISDCQ."""
    spec, prob, _ = MG.imexq_adr_case("c2")
    res = {}
    for key, scheme, nu in (("c", CISDCQ, 24), ("i", IMEXQ, 1), ("m", MISDCQ, 1)):
        o = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=2, n_sweeps=1, nu=nu, convention=1)
        res[key], _, _ = oracle.integrate(prob, spec.phi0, o)
    assert np.abs(res["c"] - res["i"]).max() <= 1e-10
    assert np.abs(res["c"] - res["m"]).max() > 1e-5


def test_oracle_coupled_iteration_cap_and_capability(oracle):
    spec, prob, o = MG.imexq_adr_case("c2")
    with pytest.raises(oracle.OracleError, match="coupled solve did not converge"):
        oracle.integrate(with_coupled(spec.problem, 1e-13, 1), spec.phi0, o)
    with pytest.raises(oracle.OracleError, match="no coupled diffusion-reaction solve"):
        oracle.integrate(spec.problem, spec.phi0, o)  # coupled_max_iter == 0: none provided


# ------------------------------------------------------------------ GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(MG.IMEXQ_ADR))
def test_gpu_imexq_adr_matches_reference_fixture(gpu, oracle, name):
    """1-D (circulant solve), 2-D and 3-D (multigrid) grids, scalar and network reactions: final state,
    sweeps, coupled solves, Newton trips and multigrid cycles equal the unmodified reference's run
    (fixture) and the oracle's, bit for bit."""
    spec, prob, o = MG.imexq_adr_case(name)
    g = api.integrate(prob, spec.phi0, o)
    check_against_fixture(name, g.final_state, *totals(g.steps))
    c, reps, incs = oracle.integrate(prob, spec.phi0, o)
    assert np.array_equal(g.final_state, c)
    assert np.allclose(np.concatenate([s.increments for s in g.steps]), incs, rtol=1e-12, atol=0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["c3", "c5"])
def test_gpu_imexq_adr_tiled_grids(gpu, oracle, name):
    """Grids on the tiled / TMA stencil walkers (the fixture's are smaller than a tile): one IMEXQ sweep,
    every stored field of the sweep state equal to the oracle's."""
    if name == "c3":
        spec = P.config_c3(scale=16, n_steps=1)  # 64 x 64
    else:
        from test_gpu_parity import c5_like
        n = (64, 16, 12)
        spec = c5_like(n, P.constant_velocity_tables((1.0, -0.5, 0.25), n))
    prob = with_coupled(spec.problem)
    M = 3
    st = api.SweepState(prob, M)
    st.initialize(spec.phi0)
    cnt = api.SolveCounters()
    api.run_sweep(IMEXQ, st, spec.dt, 1, counters=cnt)
    orc = oracle.State(oracle.Problem(prob), M)
    orc.initialize(spec.phi0)
    orc.sweep(IMEXQ, oracle.make_tables(M, 0), spec.dt, 1)
    assert cnt.coupled == M and cnt.diffusion == 0 and cnt.reaction == 0
    for which in (_abi.FIELD_PHI, _abi.FIELD_FA, _abi.FIELD_FD, _abi.FIELD_FR, _abi.FIELD_PHI_AD):
        for m in range(1, M + 1):
            assert np.array_equal(st.field(which, m), orc.field(which, m)), (which, m)
    st.close()


@pytest.mark.gpu
def test_gpu_coupled_stage_solve_adr(gpu, oracle):
    """solve_coupled through the stage API == the oracle's, bitwise, with the same inner work."""
    spec, prob, _ = MG.imexq_adr_case("c3")
    gp = api.GpuProblem(prob, M=2)
    orc = oracle.Problem(prob)
    for coef in (0.0, 0.3 * spec.dt, 2.0 * spec.dt):
        assert np.array_equal(gp.solve_coupled(coef, spec.phi0), orc.solve(_abi.STAGE_COUPLED, coef, spec.phi0)), coef
    gp.close()


@pytest.mark.gpu
def test_gpu_cisdcq_inner_iterations_reach_imexq_adr(gpu):
    """test_integrators.cpp:195-213 on the GPU engine and the PDE class."""
    spec, prob, _ = MG.imexq_adr_case("c2")
    res = {}
    for key, scheme, nu in (("c", CISDCQ, 24), ("i", IMEXQ, 1), ("m", MISDCQ, 1)):
        o = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=2, n_sweeps=1, nu=nu, convention=1)
        res[key] = api.integrate(prob, spec.phi0, o).final_state
    assert np.abs(res["c"] - res["i"]).max() <= 1e-10
    assert np.abs(res["c"] - res["m"]).max() > 1e-5


@pytest.mark.gpu
def test_gpu_coupled_errors_match_oracle(gpu, oracle):
    """The iteration cap raises the oracle's SolveError text (step / sweep prefix included); a problem
    without the coupled stage raises the reference's CapabilityError from the sweep."""
    spec, prob, o = MG.imexq_adr_case("c2")
    capped = with_coupled(spec.problem, 1e-13, 1)
    try:
        oracle.integrate(capped, spec.phi0, o)
        raise AssertionError("the oracle converged in one iteration")
    except oracle.OracleError as e:
        want = str(e).split("] ", 1)[1]
    with pytest.raises(api.SolveError) as ge:
        api.integrate(capped, spec.phi0, o)
    assert str(ge.value) == want, (str(ge.value), want)
    # integrate wraps every sweep exception as SolveError (integrators.cpp:318-321); the sweep itself
    # raises the reference's CapabilityError
    with pytest.raises(api.SolveError, match="imexq_sweep: problem provides no coupled diffusion-reaction solve"):
        api.integrate(spec.problem, spec.phi0, o)
    st = api.SweepState(spec.problem, 2)
    st.initialize(spec.phi0)
    with pytest.raises(api.CapabilityError, match="coupled"):
        api.run_sweep(IMEXQ, st, spec.dt, 1)
    st.close()
    # the context stays usable after the failure
    g = api.integrate(prob, spec.phi0, o)
    c, _, _ = oracle.integrate(prob, spec.phi0, o)
    assert np.array_equal(g.final_state, c)
