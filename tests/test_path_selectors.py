"""Every kernel-path selector of the engine, forced one at a time, against the oracle (bitwise).

The library picks a kernel per grid shape (pair / tiled / TMA walkers, row kernels, single-block coarse
levels, graph-replayed cycles, the fused Newton + rhs kernel, ...); each choice can be overridden by an
environment variable so that the alternative path runs on a grid where it is not the default.  Most
are read once per process, so every case runs in its own interpreter: a 2-D multigrid hierarchy (C3 at
64^2), a 3-D whole-tile grid (the C5 network at 64 x 16 x 12) and a ragged 3-D grid (30 x 12 x 9), one
MISDCQ and one concurrent CISDCQ step each, final state and Newton / multigrid work equal to the oracle's.
"""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, ROOT); sys.path.insert(0, ROOT + "/oracle"); sys.path.insert(0, ROOT + "/tests")
import numpy as np
import oracle
from paper_1801_01201_b200 import api, problems as P
from test_gpu_parity import c5_like
oracle.build_oracle()
specs = [P.config_c3(scale=16, n_steps=1)]
for n in ((64, 16, 12), (30, 12, 9)):
    specs.append(c5_like(n, P.constant_velocity_tables((1.0, -0.5, 0.25), n)))
for spec in specs:
    for scheme, workers in ((1, 0), (2, 2)):
        o = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=3, n_sweeps=2, nu=1, workers=workers)
        g = api.integrate(spec.problem, spec.phi0, o)
        c, reps, _ = oracle.integrate(spec.problem, spec.phi0, o)
        assert np.array_equal(g.final_state, c), (spec.problem.n, scheme)
        assert g.steps[0].counters.newton_iterations == reps[0].counters.newton_iterations, (spec.problem.n, scheme)
        assert g.steps[0].counters.mg_cycles == reps[0].counters.mg_cycles, (spec.problem.n, scheme)
print("selector ok")
"""

SELECTORS = [
    ("CISDC_EVAL_PAIR", "0"),         # F_A/F_D: one cell per thread instead of the pair walker
    ("CISDC_EVAL_TMA", "0"),          # F_A/F_D: cp.async pair walker instead of TMA planes
    ("CISDC_FUSE_RHS", "0"),          # CISDCQ: separate k_rhs instead of the fused Newton + next rhs kernel
    ("CISDC_MG_CHECKONLY", "0"),      # multigrid: fused check + sweep instead of the residual-only last check
    ("CISDC_MG_COARSE", "0"),         # multigrid: one launch per coarse level instead of the single-block kernel
    ("CISDC_MG_GRAPHS", "0"),         # multigrid: every cycle enqueued instead of graph replays
    ("CISDC_MG_LOOP", "1"),           # multigrid: device-looped solves (WHILE graph nodes)
    ("CISDC_MG_PAIR", "0"),           # multigrid 3-D: one cell per thread
    ("CISDC_MG_PROLONG_PAIR", "0"),   # multigrid transfers: per-point kernels
    ("CISDC_MG_ROWS", "0"),           # multigrid 2-D: per-point sweeps instead of the row kernels
    ("CISDC_MG_TMA", "0"),            # multigrid 3-D: cp.async walker instead of TMA planes
    ("CISDC_RTC", "0"),               # Newton: generic dense kernel instead of the NVRTC-specialised one
    ("CISDC_STEP_GRAPH", "0"),        # steps enqueued directly instead of whole-step graph replays
]


@pytest.mark.parametrize("var,value", SELECTORS)
def test_forced_path_is_bitwise_equal_to_oracle(gpu, oracle, var, value):
    env = dict(os.environ)
    env[var] = value
    r = subprocess.run([sys.executable, "-c", "ROOT = %r\n" % ROOT + SCRIPT], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0 and "selector ok" in r.stdout, (var, value, r.stdout[-2000:], r.stderr[-4000:])
