"""Golden fixtures produced by the unmodified reference (tests/golden/make_golden.py): the CPU oracle
and the GPU engine must reproduce them bit for bit (no /root/reference needed at test time)."""
import os

import numpy as np
import pytest

from paper_1801_01201_b200 import api, problems as P

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
import sys  # noqa: E402

sys.path.insert(0, HERE)
import make_golden as MG  # noqa: E402


def load(name):
    return np.load(os.path.join(HERE, name))


def test_tables_golden(oracle):
    g = load("tables.npz")
    for M in range(1, 9):
        for conv in (0, 1):
            assert bytes(oracle.make_tables(M, conv)) == g[f"M{M}_c{conv}"].tobytes()
            assert bytes(api.make_quadrature_tables(M, conv).c) == g[f"M{M}_c{conv}"].tobytes()


def _gate(run):
    g = load("gate_c0.npz")
    spec = P.config_c0(n_x=64, n_steps=3)
    assert np.array_equal(spec.phi0, g["phi0"])
    for s, nu, c in MG.GATE_RUNS:
        o = api.IntegrateOptions(scheme=s, dt=0.05, n_steps=3, M=4, n_sweeps=4, nu=nu, convention=c)
        f, counts, incs = run(spec, o)
        k = f"s{s}_nu{nu}_c{c}"
        assert np.array_equal(f, g[k + "_final"]), k
        assert np.array_equal(counts, g[k + "_counts"]), k
        yield k, incs, g[k + "_incs"]


def test_gate_golden_oracle(oracle):
    def run(spec, o):
        f, reps, incs = oracle.integrate(spec.problem, spec.phi0, o)
        return f, np.array([[r.sweeps, r.counters.diffusion, r.counters.reaction] for r in reps]), incs

    for k, incs, ginc in _gate(run):
        assert np.array_equal(incs, ginc), k


@pytest.mark.gpu
def test_gate_golden_gpu(gpu):
    def run(spec, o):
        r = api.integrate(spec.problem, spec.phi0, o)
        counts = np.array([[s.sweeps, s.counters.diffusion, s.counters.reaction] for s in r.steps])
        return r.final_state, counts, np.concatenate([s.increments for s in r.steps])

    for k, incs, ginc in _gate(run):
        # increment_norm: the GPU's fixed-tree sum differs from the serial sum by rounding only
        assert np.allclose(incs, ginc, rtol=1e-12, atol=0), k


def _periodic(run):
    g = load("periodic.npz")
    for name in MG.PERIODIC:
        spec, schemes = MG.periodic_runs(name)
        assert np.array_equal(spec.phi0, g[f"{name}_phi0"])
        for s in schemes:
            o = api.IntegrateOptions(scheme=s, dt=spec.dt, n_steps=spec.n_steps, M=spec.M, n_sweeps=spec.n_sweeps,
                                     nu=1)
            f, newton, mg, sweeps, incs = run(spec, o)
            k = f"{name}_s{s}"
            assert np.array_equal(f, g[k + "_final"]), k
            c = g[k + "_counts"]
            assert newton == c[0] and mg == c[1] and list(sweeps) == list(c[2:]), k
            yield k, incs, g[k + "_incs"]


def test_periodic_golden_oracle(oracle):
    def run(spec, o):
        f, reps, incs = oracle.integrate(spec.problem, spec.phi0, o)
        return (f, sum(r.counters.newton_iterations for r in reps), sum(r.counters.mg_cycles for r in reps),
                [r.sweeps for r in reps], incs)

    for k, incs, ginc in _periodic(run):
        assert np.array_equal(incs, ginc), k


@pytest.mark.gpu
def test_periodic_golden_gpu(gpu):
    def run(spec, o):
        r = api.integrate(spec.problem, spec.phi0, o)
        return (r.final_state, sum(s.counters.newton_iterations for s in r.steps),
                sum(s.counters.mg_cycles for s in r.steps), [s.sweeps for s in r.steps],
                np.concatenate([s.increments for s in r.steps]))

    for k, incs, ginc in _periodic(run):
        assert np.allclose(incs, ginc[: len(incs)], rtol=1e-12, atol=0), k
