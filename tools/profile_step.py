"""One SDC time step of a config through the C-ABI (device-resident), for ncu captures.

  python tools/profile_step.py --config c5 --scale 2 [--steps 1]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1801_01201_b200 import _abi, api, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--scale", type=int, default=2)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--workers", type=int, default=2)
    ap.add_argument("--scheme", type=int, default=None)
    a = ap.parse_args()
    spec = problems.CONFIGS[a.config](scale=a.scale)
    scheme = spec.scheme if a.scheme is None else a.scheme
    opt = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps,
                               nu=spec.nu, workers=a.workers if scheme == 2 else 0)
    ctx = api.GpuContext(spec.problem, spec.M)
    for _ in range(a.steps):
        r = api.integrate(spec.problem, spec.phi0, opt, ctx=ctx)
    print("ok", a.config, spec.problem.dim, r.steps[0].counters, float(np.max(np.abs(r.final_state))))
    ctx.close()


if __name__ == "__main__":
    main()
