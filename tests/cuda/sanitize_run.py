"""One small integrate per kernel family, run under compute-sanitizer by tests/test_sanitizer.py.

  python tests/cuda/sanitize_run.py c2|c3|c5
c2: 1-D (4096 cells): cluster scan solve (DSMEM), 1-D stencils, scalar Newton.
c3: 2-D 128^2 x 3: warp-private row rings (k_eval_ad2_rows, k_mg2_rows), multigrid levels, NVRTC Newton.
c5: 3-D 64^3 x 9: cp.async plane rings (k_eval_ad3_pair, k_mg3_pair), the coarse-level kernel,
    the 9-species NVRTC Newton + dense fixup, both PMISDC streams.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_1801_01201_b200 import api, problems as P  # noqa: E402

name = sys.argv[1]
if name == "c2":
    spec, schemes = P.config_c2(scale=16, n_steps=1), ((1, 0), (2, 2))
elif name == "c3":
    spec, schemes = P.config_c3(scale=8, n_steps=1), ((1, 0), (2, 2))
else:
    spec, schemes = P.config_c5(scale=4, n_steps=1), ((2, 2),)
for scheme, workers in schemes:
    o = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=1, nu=1, workers=workers,
                             convention=spec.convention)
    r = api.integrate(spec.problem, spec.phi0, o)
    assert r.steps[0].sweeps == 1
print("sanitize_run ok", name)
