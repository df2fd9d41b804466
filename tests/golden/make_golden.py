"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures travel with the repo; tests/test_golden.py checks the oracle (CPU) and the GPU engine
against them without needing /root/reference.

  tables.npz      cisdc::make_quadrature_tables(M, convention), M = 1..8, both conventions
  gate_c0.npz     cisdc::integrate on the reference's own Dirichlet PDE (n_x = 64, a = 1, d = 2, r = 4,
                  dt = 0.05, M = 4, 3 steps x 4 sweeps): misdc, misdcq, cisdcq nu = 1/3, both conventions
  periodic.npz    the reference integrators driving the periodic ADR problem class (configs 1-5 at
                  reduced size): final state, increments, solve / Newton / multigrid counts
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import oracle as O  # noqa: E402
from paper_1801_01201_b200 import api, problems as P  # noqa: E402

GATE_RUNS = [(s, nu, c) for s, nu in ((0, 1), (1, 1), (2, 1), (2, 3)) for c in (0, 1)]
PERIODIC = {
    "c1": lambda: P.config_c1(scale=4),
    "c2": lambda: P.config_c2(scale=128, n_steps=2),
    "c3": lambda: P.config_c3(scale=32, n_steps=1),
    "c4": lambda: P.config_c4(scale=64, n_steps=1),
    "c5": lambda: P.config_c5(scale=32),
}


def periodic_runs(name):
    spec = PERIODIC[name]()
    schemes = (0, 1, 2) if name != "c5" else (1, 2)
    return spec, schemes


def main():
    if O.ref_lib() is None:
        raise SystemExit("oracle/_ref not available: build it with make -C oracle ref (needs /root/reference)")
    out = {}
    for M in range(1, 9):
        for conv in (0, 1):
            t = O.ref_make_tables(M, conv)
            out[f"M{M}_c{conv}"] = np.frombuffer(bytes(t), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "tables.npz"), **out)

    gate = {}
    spec = P.config_c0(n_x=64, n_steps=3)
    gate["phi0"] = spec.phi0
    for s, nu, c in GATE_RUNS:
        o = api.IntegrateOptions(scheme=s, dt=0.05, n_steps=3, M=4, n_sweeps=4, nu=nu, convention=c)
        f, reps, incs = O.ref_integrate(spec.problem, spec.phi0, o)
        k = f"s{s}_nu{nu}_c{c}"
        gate[k + "_final"] = f
        gate[k + "_incs"] = incs
        gate[k + "_counts"] = np.array([[r.sweeps, r.counters.diffusion, r.counters.reaction] for r in reps])
    np.savez_compressed(os.path.join(HERE, "gate_c0.npz"), **gate)

    per = {}
    for name in PERIODIC:
        spec, schemes = periodic_runs(name)
        per[f"{name}_phi0"] = spec.phi0
        for s in schemes:
            o = api.IntegrateOptions(scheme=s, dt=spec.dt, n_steps=spec.n_steps, M=spec.M, n_sweeps=spec.n_sweeps,
                                     nu=1)
            f, reps, incs = O.ref_integrate(spec.problem, spec.phi0, o)
            k = f"{name}_s{s}"
            per[k + "_final"] = f
            per[k + "_incs"] = incs
            per[k + "_counts"] = np.array([reps[0].counters.newton_iterations, reps[0].counters.mg_cycles] +
                                          [r.sweeps for r in reps])
    np.savez_compressed(os.path.join(HERE, "periodic.npz"), **per)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
