"""Parity at the BASELINE configurations' FULL sizes.

tests/golden/full_<cfg>.json are written by ``tests/golden/make_golden.py --full`` from the UNMODIFIED
reference (oracle/_ref: cisdc::integrate / cisdc::execute_pipelined driving the oracle problem
class) at the sizes the bench runs: C3 1024^2 x 3 (misdc, misdcq, cisdcq), C4 2048^2 x 9 (misdc,
misdcq, cisdcq), C5 256^3 x 9 (cisdcq nu = 1, the bench workload), one time step each.  The states
are too large to commit; the fixtures hold the sha256 of the initial and final state bytes, the
per-step counts (sweeps, diffusion / reaction solves, Newton trips, multigrid cycles) and the
increments.  The GPU must reproduce the final state BIT FOR BIT (same hash) with equal counts.
"""
import glob
import hashlib
import json
import os

import numpy as np
import pytest

from paper_1801_01201_b200 import api, problems as P

HERE = os.path.dirname(os.path.abspath(__file__))
FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "full_*.json")))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def load(path):
    with open(path) as f:
        return json.load(f)


def test_full_fixtures_present_and_consistent():
    """The committed full-size fixtures exist for C3, C4, C5 and their counts obey the schemes'
    solve counts (reference test_integrators.cpp:304-324: M solves per stage per sweep, nu M for
    CISDCQ)."""
    names = {load(p)["config"] for p in FIXTURES}
    assert {"c3", "c4", "c5"} <= names, names
    for p in FIXTURES:
        fx = load(p)
        for s, run in fx["runs"].items():
            per = fx["M"] * fx["nu"] if int(s) == 2 else fx["M"]
            assert run["sweeps"] == fx["n_sweeps"]
            assert run["diffusion"] == run["reaction"] == per * fx["n_sweeps"]
            assert run["newton_iterations"] > 0 and len(run["increments"]) == run["sweeps"]


def test_full_c3_initial_state_hash():
    """The seeded generator reproduces the fixture's initial state on this host (C3: cheap)."""
    fx = load(os.path.join(HERE, "golden", "full_c3.json"))
    assert sha(P.config_c3(n_steps=1).phi0) == fx["phi0_sha256"]


@pytest.mark.gpu
@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p)[5:-5] for p in FIXTURES])
def test_full_size_step_bitwise_vs_reference(gpu, path):
    fx = load(path)
    spec = P.CONFIGS[fx["config"]](n_steps=1)
    assert sha(spec.phi0) == fx["phi0_sha256"], "initial state differs from the fixture's (generator drift)"
    ctx = api.GpuContext(spec.problem, spec.M, spec.convention)
    try:
        for s, run in fx["runs"].items():
            s = int(s)
            for workers in ((0, 2) if s == 2 else (0,)):
                o = api.IntegrateOptions(scheme=s, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps, nu=1,
                                         workers=workers, convention=spec.convention)
                g = api.integrate(spec.problem, spec.phi0, o, ctx=ctx)
                rep = g.steps[0]
                tag = f"{fx['config']} {run['scheme']} workers={workers}"
                assert (rep.sweeps, rep.counters.diffusion, rep.counters.reaction) == (
                    run["sweeps"], run["diffusion"], run["reaction"]), tag
                assert rep.counters.newton_iterations == run["newton_iterations"], tag
                assert rep.counters.mg_cycles == run["mg_cycles"], tag
                assert sha(g.final_state) == run["final_sha256"], tag + ": final state not bit-identical"
                assert float(np.max(g.final_state)).hex() == run["final_norms"]["max"], tag
                # increments: fixed-tree device sum vs the reference's sequential sum (round-off only)
                ref_inc = np.array([float.fromhex(x) for x in run["increments"]])
                assert np.allclose(rep.increments, ref_inc, rtol=1e-12, atol=0), tag
                del g
    finally:
        ctx.close()
