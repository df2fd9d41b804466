"""GPU (native engine, through the C-ABI) against the CPU oracle and the unmodified reference.

Bar (north_star): per-step max relative state difference <= 1e-10 with identical sweep and Newton
iteration counts.  By construction (same operation order, no FMA) the engine is bit-identical to the
oracle, so most checks assert array equality; the tolerance is asserted as well.
"""
import numpy as np
import pytest

from paper_1801_01201_b200 import _abi, api, problems as P

pytestmark = pytest.mark.gpu
TOL = 1e-10


def relerr(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def opts(spec, scheme, steps=None, nu=None, workers=0, conv=None, sweeps=None):
    return api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=steps or spec.n_steps, M=spec.M,
                                n_sweeps=sweeps or spec.n_sweeps, nu=nu or spec.nu, workers=workers,
                                convention=spec.convention if conv is None else conv)


def per_step_compare(oracle, spec, scheme, steps, nu=1, workers=0, conv=0):
    """integrate step by step (n_steps = 1 fed back == one multi-step call, integrators.cpp:312-330)."""
    ctx = api.GpuContext(spec.problem, spec.M, conv)
    phi_g = spec.phi0.copy()
    phi_c = spec.phi0.copy()
    worst = 0.0
    try:
        for _ in range(steps):
            o = opts(spec, scheme, steps=1, nu=nu, workers=workers, conv=conv)
            g = api.integrate(spec.problem, phi_g, o, ctx=ctx)
            c, reps, incs = oracle.integrate(spec.problem, phi_c, o)
            worst = max(worst, relerr(g.final_state, c))
            assert g.steps[0].sweeps == reps[0].sweeps
            assert g.steps[0].counters.newton_iterations == reps[0].counters.newton_iterations
            assert g.steps[0].counters.mg_cycles == reps[0].counters.mg_cycles
            assert g.steps[0].counters.diffusion == reps[0].counters.diffusion
            assert g.steps[0].counters.reaction == reps[0].counters.reaction
            assert np.allclose(g.steps[0].increments, incs[: reps[0].sweeps], rtol=1e-12, atol=0)
            phi_g, phi_c = g.final_state, c
    finally:
        ctx.close()
    assert worst <= TOL
    return worst, phi_g, phi_c


# ------------------------------------------------------------------ config-0 gate: unmodified reference

@pytest.mark.parametrize("scheme,nu,workers", [(0, 1, 0), (1, 1, 0), (2, 1, 0), (2, 3, 0), (2, 1, 2), (2, 3, 2)])
@pytest.mark.parametrize("conv", [0, 1])
def test_gate_reference_pde_bitwise(gpu, oracle, scheme, nu, workers, conv):
    """The reference's own Dirichlet PDE (n_x = 200, a = 1, d = 2, r = 4): GPU == reference, bit for bit."""
    spec = P.config_c0(n_steps=5)
    o = opts(spec, scheme, steps=5, nu=nu, workers=workers, conv=conv)
    g = api.integrate(spec.problem, spec.phi0, o)
    if oracle.ref_lib() is not None:
        r, reps, incs = oracle.ref_integrate(spec.problem, spec.phi0, o)
    else:
        r, reps, incs = oracle.integrate(spec.problem, spec.phi0, o)
    assert np.array_equal(g.final_state, r)
    for s, rep in zip(g.steps, reps):
        assert s.sweeps == rep.sweeps
        assert (s.counters.diffusion, s.counters.reaction) == (rep.counters.diffusion, rep.counters.reaction)
    c, creps, _ = oracle.integrate(spec.problem, spec.phi0, o)
    assert sum(s.counters.newton_iterations for s in g.steps) == sum(x.counters.newton_iterations for x in creps)


# ------------------------------------------------------------------ BASELINE configs (scaled)

CASES = {
    "c1": (lambda: P.config_c1(), 10, (0, 1, 2)),
    "c2": (lambda: P.config_c2(scale=16), 3, (0, 1, 2)),
    "c3": (lambda: P.config_c3(scale=16, n_steps=1), 1, (0, 1, 2)),
    "c4": (lambda: P.config_c4(scale=32, n_steps=1), 1, (0, 1, 2)),
    "c5": (lambda: P.config_c5(scale=16), 1, (1, 2)),
}


@pytest.mark.parametrize("name", list(CASES))
def test_config_parity_per_step(gpu, oracle, name):
    make, steps, schemes = CASES[name]
    spec = make()
    for scheme in schemes:
        _, g, c = per_step_compare(oracle, spec, scheme, steps)
        assert np.array_equal(g, c), f"{name} scheme {scheme}: not bitwise"


def test_config1_full_run_both_schemes(gpu, oracle):
    """C1 exactly as specified: N = 256, 100 steps, MISDC and PMISDC (CISDCQ nu = 1, concurrent)."""
    spec = P.config_c1()
    for scheme, workers in ((0, 0), (2, 2)):
        o = opts(spec, scheme, workers=workers)
        g = api.integrate(spec.problem, spec.phi0, o)
        c, reps, _ = oracle.integrate(spec.problem, spec.phi0, o)
        assert relerr(g.final_state, c) <= TOL
        assert np.array_equal(g.final_state, c)
        assert sum(s.counters.newton_iterations for s in g.steps) == sum(r.counters.newton_iterations for r in reps)


@pytest.mark.parametrize("name", ["c2", "c3", "c5"])
def test_pipelined_equals_serial_and_nested_iterations(gpu, oracle, name):
    """execute_pipelined semantics: concurrent D/R streams == serial cell order, bitwise, nu = 1, 3."""
    spec = CASES[name][0]()
    for nu in (1, 3):
        a = api.integrate(spec.problem, spec.phi0, opts(spec, 2, steps=1, nu=nu, workers=0))
        b = api.integrate(spec.problem, spec.phi0, opts(spec, 2, steps=1, nu=nu, workers=2))
        c, reps, _ = oracle.integrate(spec.problem, spec.phi0, opts(spec, 2, steps=1, nu=nu))
        assert np.array_equal(a.final_state, b.final_state)
        assert np.array_equal(a.final_state, c)
        assert b.steps[0].counters.diffusion == nu * spec.M * spec.n_sweeps
        assert b.steps[0].counters.newton_iterations == reps[0].counters.newton_iterations


def test_full_size_config2_step(gpu, oracle):
    """C2 at its full size (N = 65536, 5 nodes, 8 sweeps): two steps, all three schemes."""
    spec = P.config_c2()
    for scheme in (0, 1, 2):
        per_step_compare(oracle, spec, scheme, 2)


def test_1d_direct_solve_vs_independent_banded_lu(gpu, oracle):
    """The GPU's exact circulant solve against the oracle's cyclic banded LU (reference banded_solve
    semantics, an independent algorithm): agreement to round-off at C2 size and stiffness."""
    spec = P.config_c2()
    prob = api.GpuProblem(spec.problem, M=4)
    desc_lu = P.config_c2().problem
    desc_lu.diffusion_solver = _abi.DIFFUSION_BANDED_ORACLE
    lu = oracle.Problem(desc_lu)
    rng = np.random.default_rng(7)
    rhs = spec.phi0 + 0.01 * rng.standard_normal(spec.phi0.size)
    t = api.make_quadrature_tables(4)
    for m in range(4):
        coef = spec.dt * t.QtI[m, m]
        x = prob.solve_diffusion(coef, rhs)
        y = lu.solve(_abi.STAGE_DIFFUSION, coef, rhs)
        assert relerr(x, y) <= 1e-12
    prob.close()


@pytest.mark.parametrize("name", list(CASES))
def test_stage_level_bitwise(gpu, oracle, name):
    """OperatorSplitProblem stages one by one: eval_* and solve_* == oracle."""
    spec = CASES[name][0]()
    prob = api.GpuProblem(spec.problem, M=spec.M)
    orc = oracle.Problem(spec.problem)
    x = spec.phi0
    for stage, fn in ((0, prob.eval_advection), (1, prob.eval_diffusion), (2, prob.eval_reaction)):
        assert np.array_equal(fn(x), orc.eval(stage, x)), stage
    coef = spec.dt * 0.3
    c1, c2 = api.SolveCounters(), _abi.CountersC()
    assert np.array_equal(prob.solve_diffusion(coef, x, c1), orc.solve(1, coef, x, c2))
    assert np.array_equal(prob.solve_reaction(coef, x, c1), orc.solve(2, coef, x, c2))
    assert c1.newton_iterations == c2.newton_iterations and c1.mg_cycles == c2.mg_cycles
    # coef == 0 is the identity (reaction_diffusion.cpp:159)
    assert np.array_equal(prob.solve_diffusion(0.0, x), x)
    prob.close()


def test_sweep_state_api(gpu, oracle):
    """SweepState: initialize / set_node_values / run_sweep / fields / increment == oracle state."""
    spec = P.config_c2(scale=64)
    M = spec.M
    rng = np.random.default_rng(3)
    vals = np.stack([spec.phi0 + 0.01 * rng.standard_normal(spec.phi0.size) for _ in range(M + 1)])
    st = api.SweepState(spec.problem, M)
    st.set_node_values(vals)
    fields, cnt = oracle.sweeps(spec.problem, M, 0, 1, spec.dt, 1, 3, values=vals)
    cnt_g = api.SolveCounters()
    prev = st.phi(M)
    for _ in range(3):
        api.run_sweep(api.Scheme.misdcq, st, spec.dt, 1, cnt_g)
        inc = st.increment()
        assert abs(inc - np.mean(np.abs(st.phi(M) - prev))) <= 1e-12 * max(inc, 1e-300)
        prev = st.phi(M)
    for w, get in enumerate((st.phi, st.fa, st.fd, st.fr, st.phi_ad)):
        for m in range(M + 1):
            if w == 4 and m == 0:
                continue
            assert np.array_equal(get(m), fields[w, m]), (w, m)
    assert cnt_g.newton_iterations == cnt.newton_iterations
    assert (cnt_g.diffusion, cnt_g.reaction) == (3 * M, 3 * M)
    st.close()


def test_newton_failure_reports_first_cell(gpu, oracle):
    """A diverging undamped Newton (config-4 network at dt = 5e-4) raises SolveError naming the same
    first failing cell as the oracle, with integrate's step/sweep context."""
    spec = P.config_c4(scale=64, n_steps=1)
    o = opts(spec, 1, steps=1)
    o.dt = 5e-4
    with pytest.raises(oracle.OracleError) as ce:
        oracle.integrate(spec.problem, spec.phi0, o)
    with pytest.raises(api.SolveError) as ge:
        api.integrate(spec.problem, spec.phi0, o)
    msg_c, msg_g = str(ce.value), str(ge.value)
    assert "integrate: step 1" in msg_g and "cell" in msg_g
    cell_c = msg_c.split("cell ")[1].split(":")[0]
    cell_g = msg_g.split("cell ")[1].split(":")[0]
    assert cell_c == cell_g


def test_invalid_arguments(gpu):
    spec = P.config_c1(scale=4)
    with pytest.raises(ValueError):
        api.integrate(spec.problem, spec.phi0, api.IntegrateOptions(n_sweeps=0))
    with pytest.raises(ValueError):
        api.integrate(spec.problem, spec.phi0, api.IntegrateOptions(scheme=2, nu=0, M=2, n_sweeps=1))
    st = api.SweepState(spec.problem, 2)
    st.initialize(spec.phi0)
    with pytest.raises(api.CapabilityError):
        api.run_sweep(api.Scheme.imexq, st, 1e-3)
    with pytest.raises(ValueError):
        st.initialize(np.zeros(3))
    st.close()


def test_run_to_run_determinism(gpu):
    spec = P.config_c4(scale=32, n_steps=1)
    o = opts(spec, 2, steps=1, workers=2)
    a = api.integrate(spec.problem, spec.phi0, o).final_state
    b = api.integrate(spec.problem, spec.phi0, o).final_state
    assert np.array_equal(a, b)


def test_multigrid_residual_property_full_size(gpu):
    """C3 at full size (1024^2 x 3): the diffusion solve meets its residual tolerance and is linear."""
    spec = P.config_c3()
    prob = api.GpuProblem(spec.problem, M=spec.M)
    coef = spec.dt * 0.3
    x = prob.solve_diffusion(coef, spec.phi0)
    # residual b - (x - coef F_D(x)) per species, inf-norm relative to ||b||
    r = spec.phi0 - (x - coef * prob.eval_diffusion(x))
    nc = spec.problem.ncell
    for s in range(3):
        assert np.max(np.abs(r[s * nc:(s + 1) * nc])) <= 1e-9 * np.max(np.abs(spec.phi0[s * nc:(s + 1) * nc]))
    prob.close()


def test_stop_tol_and_reports(gpu, oracle):
    spec = P.config_c2(scale=64)
    o = opts(spec, 1, steps=3, sweeps=30)
    o.stop_tol = 1e-13
    g = api.integrate(spec.problem, spec.phi0, o)
    c, reps, incs = oracle.integrate(spec.problem, spec.phi0, o)
    assert np.array_equal(g.final_state, c)
    assert [s.sweeps for s in g.steps] == [r.sweeps for r in reps]
    assert all(s.sweeps < 30 for s in g.steps)


def test_order_of_accuracy_matches_oracle(gpu, oracle):
    """The reference's refinement study (refinement.cpp:74-122, defaults of refinement.hpp:29-42:
    n_x = 200, a = 1, d = 2, r = 4, T = 0.4, dt = 0.05 .. 0.00625, reference MISDCQ at dx/32 with 8
    sweeps) run on the GPU: slopes equal the CPU oracle's within 0.05 and meet SPEC.md's acceptance
    bands (2 sweeps -> 2.0 +- 0.25, 4 sweeps -> 4.0 +- 0.4) for MISDC, MISDCQ and CISDCQ-1."""
    from paper_1801_01201_b200 import refinement as R
    opt = R.RefinementOptions(sweep_counts=(2, 4))
    g = R.refinement_study(opt)
    c = R.refinement_study(opt, integrate=oracle.integrate)
    assert np.array_equal(g.reference, c.reference)
    for cg, cc in zip(g.curves, c.curves):
        assert abs(cg.slope - cc.slope) <= 0.05
        band = 0.25 if cg.sweeps == 2 else 0.4
        assert abs(cg.slope - cg.sweeps) <= band, (cg.scheme, cg.sweeps, cg.slope)


# ------------------------------------------------------------------ 3-D tiled stencils: ragged grids, variable velocity

def c5_like(n, vel, seed=11):
    """The C5 network on an arbitrary 3-D grid (ragged against the 32 x 8 tiles and the 32-plane
    z-chunks) with the given separable face-velocity tables."""
    reac, prod, k, D = P._c45_network()
    p = P.ProblemDesc(ndim=3, n=n, nspecies=9, h=tuple(1.0 / x for x in n), vel=vel, diffusivity=D,
                      reaction_kind=_abi.REACTION_MASS_ACTION, reactants=reac, products=prod, rate_constants=k,
                      name="c5-like")
    P.mg_defaults(p, 1e-10)
    rng = np.random.default_rng(seed)
    fields = P._normalised_fields(rng, n, 9, 16, 3)
    return P.RunSpec(p, P.to_layout(fields), 2, 6, 4, 1e-5, 1, nu=1, name="c5-like", schemes=(2,))


def random_velocity_tables(n, seed=3):
    rng = np.random.default_rng(seed)
    return {(a, b): rng.uniform(0.2, 1.5, n[b]) * (1 if (a + b) % 2 else -1) for a in range(3) for b in range(3)
            if (a + b) % 3 != 1}


@pytest.mark.parametrize("n,variable", [((40, 20, 36), True), ((40, 20, 36), False), ((16, 8, 70), True),
                                         ((64, 24, 33), False), ((37, 20, 36), True), ((37, 12, 40), False)])
def test_tiled_3d_ragged_and_variable_velocity(gpu, oracle, n, variable):
    """The tiled 3-D F_A/F_D and multigrid kernels (cp.async plane ring, z carry, uniform-velocity
    specialisation; two cells per thread for even nx, one for odd nx) on grids that are not
    multiples of the tiles or the 32-plane chunk, with spatially varying (general path) or uniform
    (specialised path) face velocities: bitwise."""
    vel = random_velocity_tables(n) if variable else P.constant_velocity_tables((1.0, -0.5, 0.25), n)
    spec = c5_like(n, vel)
    for workers in (0, 2):
        _, g, c = per_step_compare(oracle, spec, 2, 1, workers=workers)
        assert np.array_equal(g, c)


# ------------------------------------------------------------------ shared-reciprocal division (newton.cuh)

def test_div_rcp_bitexact(gpu, tmp_path):
    """div_rcp(a, b, rcp_refined(b)) == IEEE a / b bit for bit (5 x 2^26 operand pairs: ordinary,
    extreme exponents, binade edges, near-midpoint quotients, zeros / infinities / NaN)."""
    import os
    import shutil
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    exe = str(tmp_path / "div_check")
    subprocess.run([nvcc, "-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false",
                    "-I", os.path.join(root, "include"), "-I", os.path.join(root, "paper_1801_01201_b200", "csrc"),
                    os.path.join(root, "tests", "cuda", "div_check.cu"), "-o", exe], check=True, capture_output=True)
    out = subprocess.run([exe, str(1 << 26)], capture_output=True, text=True, timeout=300)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr


# ------------------------------------------------------------------ PMISDC schedule trace

@pytest.mark.parametrize("nu", [1, 3])
def test_gpu_schedule_trace_valid(gpu, oracle, nu):
    """execute_pipelined on the GPU returns a ScheduleTrace (per-cell stream timestamps) that both the
    Python validator and the reference's validate_schedule_trace accept, and the state equals the
    serial cell order bitwise."""
    spec = P.config_c5(scale=16)
    st = api.SweepState(spec.problem, spec.M)
    try:
        st.initialize(spec.phi0)
        tr = api.execute_pipelined(st, spec.dt, nu, workers=2)
        piped = st.phi(spec.M)
        g = api.build_task_graph(spec.M, nu)
        assert len(tr.cells) == 2 * spec.M * nu and tr.workers == 2
        assert api.validate_schedule_trace(g, tr) == ""
        if oracle.ref_lib() is not None:
            assert oracle.ref_validate_schedule_trace(spec.M, nu, tr) == ""
        st.initialize(spec.phi0)
        api.run_sweep(api.Scheme.cisdcq, st, spec.dt, nu)
        assert np.array_equal(st.phi(spec.M), piped)
    finally:
        st.ctx.close()


# ------------------------------------------------------------------ 2-D row-streaming kernels: ragged grids

@pytest.mark.parametrize("n", [(70, 46), (130, 33), (64, 9), (71, 40)])
def test_rows_2d_ragged(gpu, oracle, n):
    """The row-streaming 2-D F_A/F_D and multigrid sweeps (even nx >= 64; odd nx takes the per-point
    kernels) with the vortex velocity, on grids ragged against the 64-column strips and the row
    chunks: bitwise equal to the oracle, all three schemes."""
    reac, prod, k, D = P._c45_network()
    p = P.ProblemDesc(ndim=2, n=(n[0], n[1], 1), nspecies=9, h=(1.0 / n[0], 1.0 / n[1], 1.0),
                      vel=P.vortex_tables(n[0], n[1]), diffusivity=D, reaction_kind=_abi.REACTION_MASS_ACTION,
                      reactants=reac, products=prod, rate_constants=k, newton_tol=1e-12, name="c4-like")
    P.mg_defaults(p)
    rng = np.random.default_rng(5)
    fields = P._normalised_fields(rng, n, 9, 16, 3)
    spec = P.RunSpec(p, P.to_layout(fields), 1, 4, 4, 1e-5, 1, name="c4-like", schemes=(0, 1, 2))
    for scheme in (0, 1, 2):
        _, g, c = per_step_compare(oracle, spec, scheme, 1)
        assert np.array_equal(g, c)


# ------------------------------------------------------------------ Newton/LU edge values (rtc.cuh deferral)

@pytest.mark.parametrize("scheme", [1, 2])
def test_newton_exact_zero_concentrations(gpu, oracle, scheme):
    """Exact zeros (+0.0 and -0.0) in the species the rates multiply by: Jacobian entries and LU
    multipliers become exact zeros, whose quotients fall outside the branch-free division's range
    test, so those cells take the exact dense path.  The state must stay bit-identical to the
    oracle (signed zeros included)."""
    n = (32, 16, 8)
    spec = c5_like(n, P.constant_velocity_tables((1.0, -0.5, 0.25), n), seed=5)
    phi = spec.phi0.reshape(9, n[2], n[1], n[0]).copy()
    reac, _, _, _ = P._c45_network()
    partners = sorted({int(b) for a, b in np.asarray(reac).reshape(-1, 2) if b >= 0})
    for q, s in enumerate(partners[:3]):
        phi[s, :, 2 + q:10 + q, 3:20] = 0.0
        phi[s, 1, 12, 5 + q] = -0.0
    spec.phi0[:] = phi.reshape(-1)
    for workers in (0, 2) if scheme == 2 else (0,):
        o = opts(spec, scheme, steps=1, workers=workers)
        g = api.integrate(spec.problem, spec.phi0, o)
        c, reps, _ = oracle.integrate(spec.problem, spec.phi0, o)
        assert np.array_equal(g.final_state.view(np.uint64), c.view(np.uint64))
        assert g.steps[0].counters.newton_iterations == reps[0].counters.newton_iterations


# ------------------------------------------------------------------ multigrid hierarchies (several levels)

def mg_levels(p, coef):
    """Levels mg_plan uses for this coefficient (the stiffness criterion of multigrid.cuh / the oracle)."""
    n = list(p.n[: p.ndim])
    L = 1
    while all(x % 2 == 0 and x // 2 >= max(p.mg_min_coarse, 4) for x in n):
        csum = sum(max(p.diffusivity) / (12.0 * (p.h[a] * 2 ** (L - 1)) ** 2) for a in range(p.ndim))
        emax = 1.0 + coef * 64.0 * csum
        if (emax - 1.0) / (emax + 1.0) <= 0.1:
            break
        n = [x // 2 for x in n]
        L += 1
    return L


@pytest.mark.parametrize("n", [(128, 96, 1), (64, 32, 1), (64, 32, 48), (256, 192, 1)])
def test_multigrid_hierarchy_bitwise(gpu, oracle, n):
    """Stiff diffusion (several multigrid levels: restriction, prolongation, coarse sweeps, the
    single-block coarse kernel) on 2-D and 3-D grids, C3's reaction chain: bitwise equal to the
    oracle with equal V-cycle counts, MISDCQ and CISDCQ (serial and concurrent)."""
    ndim = 3 if n[2] > 1 else 2
    vel = P.constant_velocity_tables((1.0, -0.5, 0.25), n) if ndim == 3 else P.vortex_tables(n[0], n[1])
    p = P.ProblemDesc(ndim=ndim, n=n, nspecies=3, h=tuple(1.0 / x for x in n[:ndim]) + (1.0,) * (3 - ndim),
                      vel=vel, diffusivity=np.array([2.0, 0.5, 0.1]), reaction_kind=_abi.REACTION_MASS_ACTION,
                      reactants=np.array([[0, -1], [1, -1], [2, -1]], dtype=np.int32),
                      products=np.array([[1, -1], [2, -1], [0, -1]], dtype=np.int32),
                      rate_constants=np.array([1.0, 1e2, 1e4]), name="mg-levels")
    P.mg_defaults(p)
    p.mg_coarse_sweeps = 4
    dt = 1e-3
    assert mg_levels(p, dt * 0.05) >= 3
    rng = np.random.default_rng(7)
    shape = n[:ndim]
    fields = [np.maximum(1.0 / 3.0 + P.random_fourier_field(rng, shape, 16, 0.1, 4), 1e-8) for _ in range(3)]
    spec = P.RunSpec(p, P.to_layout(fields), 1, 4, 2, dt, 1, name="mg-levels", schemes=(1, 2))
    for scheme, workers in ((1, 0), (2, 0), (2, 2)):
        _, g, c = per_step_compare(oracle, spec, scheme, 1, workers=workers)
        assert np.array_equal(g, c)


def _cap_problem(cap):
    n = (64, 32, 1)
    p = P.ProblemDesc(ndim=2, n=n, nspecies=3, h=(1 / 64, 1 / 32, 1.0), vel=P.vortex_tables(64, 32),
                      diffusivity=np.array([2.0, 0.5, 0.1]), reaction_kind=_abi.REACTION_MASS_ACTION,
                      reactants=np.array([[0, -1], [1, -1], [2, -1]], dtype=np.int32),
                      products=np.array([[1, -1], [2, -1], [0, -1]], dtype=np.int32),
                      rate_constants=np.array([1.0, 1e2, 1e4]), name="mg-cap")
    P.mg_defaults(p)
    p.mg_coarse_sweeps = 4
    p.mg_max_cycles = cap
    return p


@pytest.mark.parametrize("cap", [17, 18, 19, 20, 21])
def test_multigrid_cycle_cap_matches_oracle(gpu, oracle, cap):
    """mg_max_cycles near the solves' cycle counts (multigrid.cuh cap path): a solve that
    needs more than the cap must fail exactly where the oracle fails (same step, sweep, species and
    cycle count in the message), including the sweeps where an earlier solve with the same coefficient
    predicted a shorter batch (cap 18 / CISDCQ fails in sweep 4, cap 20 / MISDC in sweep 2); a run
    within the cap is bitwise equal."""
    rng = np.random.default_rng(1)
    phi0 = np.abs(1 / 3 + 0.1 * rng.standard_normal(64 * 32 * 3))
    for scheme in (0, 1, 2):
        o = api.IntegrateOptions(scheme=scheme, dt=1e-3, n_steps=2, M=4, n_sweeps=4, nu=1)
        try:
            c, reps, _ = oracle.integrate(_cap_problem(cap), phi0, o)
            cerr = None
        except oracle.OracleError as e:
            cerr = str(e)
        try:
            g = api.integrate(_cap_problem(cap), phi0, o)
            gerr = None
        except api.SolveError as e:
            gerr = str(e)
        if cerr is None:
            assert gerr is None, gerr
            assert np.array_equal(g.final_state, c)
            assert [s.counters.mg_cycles for s in g.steps] == [r.counters.mg_cycles for r in reps]
        else:
            assert gerr is not None, f"cap {cap} scheme {scheme}: GPU succeeded where the oracle failed: {cerr}"
            # oracle: "[3] integrate: step s, sweep k: solve_diffusion: multigrid: species i: no convergence
            # in N cycles (residual ..., target ...)"
            want = cerr.split("] ", 1)[1].split(" (residual")[0]
            assert gerr == want, (gerr, want)


def test_c2_end_to_end_vs_independent_banded_lu(gpu, oracle):
    """C2 at its full size (N = 65536), 2 steps, every scheme: the GPU's exact circulant scan against
    the oracle driven with the INDEPENDENT 1-D solver (the ring folded into a band and solved by the
    restated banded_solve, reference linalg.cpp:105-155) -- not the emulation of the GPU's blocked scan.
    Bar (north_star): per step max relative difference <= 1e-10.  The two 1-D solvers differ in
    round-off (<= 1e-12, test_1d_direct_solve_vs_independent_banded_lu), so a few of the 65536 x 5 x 8
    cell solves per step whose residual lands next to the Newton tolerance take one trip more or less:
    the Newton-iteration counts must agree to 1e-6 relative (measured: 2 trips in 9.4 million).  Equal
    counts, bit for bit, are pinned against the oracle that runs the GPU's own scan order
    (test_config_parity_per_step)."""
    spec = P.config_c2(n_steps=2)
    lu = P.config_c2(n_steps=2).problem
    lu.diffusion_solver = _abi.DIFFUSION_BANDED_ORACLE
    for scheme in (0, 1, 2):
        phi_g = spec.phi0.copy()
        phi_c = spec.phi0.copy()
        for step in range(2):
            o = opts(spec, scheme, steps=1)
            g = api.integrate(spec.problem, phi_g, o)
            c, reps, _ = oracle.integrate(lu, phi_c, o)
            err = relerr(g.final_state, c)
            assert err <= TOL, (scheme, step, err)
            ng, nc = g.steps[0].counters.newton_iterations, reps[0].counters.newton_iterations
            assert abs(ng - nc) <= 1e-6 * nc, (scheme, step, ng, nc)
            assert g.steps[0].sweeps == reps[0].sweeps
            phi_g, phi_c = g.final_state, c


@pytest.mark.parametrize("scheme", [1, 2])
def test_rhs_exact_zero_skip_with_wild_values(gpu, oracle, scheme):
    """k_rhs skips the F_A reads of terms whose cE is an exact zero (literal convention) unless an F_A
    evaluation flagged a value >= 2^1022 / Inf / NaN (Ops::wild).  A state with one huge value
    (F_A overflows there) must still give the oracle's outcome: the same error, or the same bits
    (NaN positions included)."""
    spec = P.config_c3(scale=16, n_steps=1)
    phi0 = spec.phi0.copy()
    phi0[1000] = 1e306
    o = opts(spec, scheme, steps=1)
    try:
        c, reps, _ = oracle.integrate(spec.problem, phi0, o)
        cerr = None
    except oracle.OracleError as e:
        cerr = str(e)
    try:
        g = api.integrate(spec.problem, phi0, o)
        gerr = None
    except api.SolveError as e:
        gerr = str(e)
    if cerr is None:
        assert gerr is None, gerr
        assert np.array_equal(g.final_state, c, equal_nan=True)
    else:
        assert gerr is not None
        assert cerr.split("] ", 1)[1].split(" (residual")[0] == gerr


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_device_looped_multigrid_bitwise(gpu, oracle, name, monkeypatch):
    """CISDC_MG_LOOP=1: every multigrid solve is one CUDA graph whose WHILE node runs the V-cycles until
    the decision kernel (k_mg_update_loop) stops it -- no host synchronisation per solve.  Same cycles,
    same bits and counts as the oracle (and as the host-driven loop)."""
    monkeypatch.setenv("CISDC_MG_LOOP", "1")
    make, steps, schemes = CASES[name]
    spec = make()
    for scheme in schemes:
        _, g, c = per_step_compare(oracle, spec, scheme, steps)
        assert np.array_equal(g, c), f"{name} scheme {scheme}: not bitwise"


@pytest.mark.parametrize("cap", [17, 18, 20])
def test_device_looped_multigrid_cap(gpu, oracle, cap, monkeypatch):
    """The cycle cap inside the device loop: the decision kernel flags the failure and ends the WHILE
    loop; the error text equals the oracle's, a run within the cap is bitwise equal."""
    monkeypatch.setenv("CISDC_MG_LOOP", "1")
    test_multigrid_cycle_cap_matches_oracle(gpu, oracle, cap)


@pytest.mark.parametrize("n,variable", [((64, 24, 33), False), ((128, 16, 40), False), ((64, 8, 9), False),
                                         ((64, 16, 38), True), ((128, 8, 13), True), ((192, 24, 64), False)])
def test_tma_staged_multigrid_sweeps(gpu, oracle, n, variable, monkeypatch):
    """Whole-tile 3-D grids (nx % 64 == 0, ny % 8 == 0) run the level-0 multigrid sweeps and checks and
    the F_A/F_D evaluation on the TMA walker (tma.cuh: five bulk-tensor boxes per plane, mbarrier
    completion, plane loop unrolled by the ring size); the cp.async walkers are forced with
    CISDC_MG_TMA=0 / CISDC_EVAL_TMA=0.  Chunk lengths of 32 planes and ragged tails (33, 38, 40, 13, 9,
    64 planes), uniform and variable face velocities.  Both bitwise equal to the oracle (and so to
    each other)."""
    vel = random_velocity_tables(n) if variable else P.constant_velocity_tables((1.0, -0.5, 0.25), n)
    spec = c5_like(n, vel)
    runs = []
    for flag in ("1", "0"):
        monkeypatch.setenv("CISDC_MG_TMA", flag)
        monkeypatch.setenv("CISDC_EVAL_TMA", flag)
        _, g, c = per_step_compare(oracle, spec, 2, 1, workers=2)
        assert np.array_equal(g, c)
        runs.append(g)
    assert np.array_equal(runs[0], runs[1])


@pytest.mark.parametrize("case", ["c0", "c1", "c2", "linear"])
def test_step_graph_replay_bitwise(gpu, oracle, case, monkeypatch):
    """Steps without host decisions inside (no stop tolerance, no host-synchronised multigrid) are
    captured once as a CUDA graph and replayed (the first step of a context runs directly): the
    final state, per-step sweeps, stage counts, Newton counts and increments equal both the direct
    enqueue (CISDC_STEP_GRAPH=0) and the oracle, over several steps and every scheme."""
    if case == "c0":
        spec, schemes = P.config_c0(n_steps=4), ((0, 1), (1, 1), (2, 3))
    elif case == "c1":
        spec, schemes = P.config_c1(), ((0, 1), (2, 1))
    elif case == "c2":
        spec, schemes = P.config_c2(scale=16, n_steps=3), ((1, 1), (2, 1))
    else:
        p = P.linear_scalar(0.5, -40.0, -3.0, batch=4097)
        spec = P.RunSpec(p, np.linspace(-1.0, 1.0, 4097), 3, 3, 4, 0.05, 3, name="linear")
        schemes = ((3, 1), (2, 2))
    for scheme, nu in schemes:
        res = {}
        for flag in ("1", "0"):
            monkeypatch.setenv("CISDC_STEP_GRAPH", flag)
            o = opts(spec, scheme, steps=min(spec.n_steps, 6), nu=nu, workers=2 if scheme == 2 else 0)
            ctx = api.GpuContext(spec.problem, spec.M, spec.convention)
            try:
                api.integrate(spec.problem, spec.phi0, o, ctx=ctx)  # the context's first step runs directly
                res[flag] = api.integrate(spec.problem, spec.phi0, o, ctx=ctx)
            finally:
                ctx.close()
        c, reps, incs = oracle.integrate(spec.problem, spec.phi0, o)
        g, d = res["1"], res["0"]
        assert np.array_equal(g.final_state, d.final_state) and np.array_equal(g.final_state, c)
        for a, b, r in zip(g.steps, d.steps, reps):
            assert a.sweeps == b.sweeps == r.sweeps
            assert (a.counters.diffusion, a.counters.reaction, a.counters.coupled, a.counters.newton_iterations) == \
                (r.counters.diffusion, r.counters.reaction, r.counters.coupled, r.counters.newton_iterations)
            assert np.array_equal(a.increments, b.increments)


def test_step_graph_failure_reports_like_direct(gpu, oracle, monkeypatch):
    """A Newton failure inside a replayed step reports the oracle's message (the tags of the captured
    enqueue are restored on every replay)."""
    spec = P.config_c1(scale=1)
    spec.problem.newton_max_iter = 1  # every cell hits the cap
    o = opts(spec, 0, steps=1)
    with pytest.raises(oracle.OracleError) as ce:
        oracle.integrate(spec.problem, spec.phi0, o)
    want = str(ce.value).split("] ", 1)[1]
    ctx = api.GpuContext(spec.problem, spec.M, spec.convention)
    try:
        for _ in range(3):  # direct, captured, replayed
            with pytest.raises(api.SolveError) as ge:
                api.integrate(spec.problem, spec.phi0, o, ctx=ctx)
            assert str(ge.value) == want
    finally:
        ctx.close()
