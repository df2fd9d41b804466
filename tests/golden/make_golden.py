"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures travel with the repo; tests/test_golden.py checks the oracle (CPU) and the GPU engine
against them without needing /root/reference.

  tables.npz      cisdc::make_quadrature_tables(M, convention), M = 1..8, both conventions
  gate_c0.npz     cisdc::integrate on the reference's own Dirichlet PDE (n_x = 64, a = 1, d = 2, r = 4,
                  dt = 0.05, M = 4, 3 steps x 4 sweeps): misdc, misdcq, cisdcq nu = 1/3, both conventions
  periodic.npz    the reference integrators driving the periodic ADR problem class (configs 1-5 at
                  reduced size): final state, increments, solve / Newton / multigrid counts
  imexq_adr.npz   (--imexq writes only this one) the reference's imexq_sweep driving the periodic ADR class's
                  coupled stage (configs 1, 2, 3, 5 at reduced size): final state, increments, per-step
                  sweeps / coupled solves / Newton trips / multigrid cycles
  full_<cfg>.json (--full [c3 c4 c5]) the same at the BASELINE configs' FULL sizes, one time step:
                  C3 1024^2 x 3 (misdc, misdcq, cisdcq), C4 2048^2 x 9 (misdc, misdcq, cisdcq),
                  C5 256^3 x 9 (cisdcq nu = 1 through execute_pipelined, the bench workload).  The
                  states are too large to commit, so the fixture holds the sha256 of the initial and
                  final state bytes, per-step counts (sweeps, D/R solves, Newton trips, multigrid
                  cycles), the increments and a few norms (hex floats), plus the run's host, threads
                  and wall time.  C5 needs ~100 GB of host RAM (the reference's SweepState layout):
                  generate it on the GPU box's host (196 GB), e.g.
                    CISDC_ORACLE_THREADS=16 python tests/golden/make_golden.py --full c5
                  (the oracle problem class's per-cell loops are threaded; results are bit-identical
                  at any thread count, see oracle/co_problems.c).
"""
import hashlib
import json
import os
import platform
import sys
import time

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


FULL = {
    "c3": (lambda: P.config_c3(n_steps=1), (0, 1, 2)),
    "c4": (lambda: P.config_c4(n_steps=1), (0, 1, 2)),
    "c5": (lambda: P.config_c5(n_steps=1), (2,)),
}


# IMEXQ on the periodic ADR class (its coupled stage, cisdc_gpu.h): the unmodified imexq_sweep
# (integrators.cpp:145-173) driving AdrProblem::solve_coupled; (config, M, sweeps, steps)
IMEXQ_ADR = {
    "c1": (lambda: P.config_c1(scale=4), 3, 3, 2),
    "c2": (lambda: P.config_c2(scale=128, n_steps=2), 3, 3, 2),
    "c3": (lambda: P.config_c3(scale=32, n_steps=1), 3, 2, 1),
    "c5": (lambda: P.config_c5(scale=32), 2, 2, 1),
}


def imexq_adr_case(name):
    import dataclasses
    make, M, sweeps, steps = IMEXQ_ADR[name]
    spec = make()
    prob = dataclasses.replace(spec.problem, coupled_tol=1e-13, coupled_max_iter=60)
    o = api.IntegrateOptions(scheme=3, dt=spec.dt, n_steps=steps, M=M, n_sweeps=sweeps, nu=1)
    return spec, prob, o


def imexq_adr():
    out = {}
    for name in IMEXQ_ADR:
        spec, prob, o = imexq_adr_case(name)
        f, reps, incs = O.ref_integrate(prob, spec.phi0, o)
        out[f"{name}_phi0"] = spec.phi0
        out[f"{name}_final"] = f
        out[f"{name}_incs"] = incs
        out[f"{name}_counts"] = np.array([[r.sweeps, r.counters.coupled, r.counters.newton_iterations,
                                           r.counters.mg_cycles] for r in reps])
        print("imexq", name, prob.n, out[f"{name}_counts"].tolist(), flush=True)
    np.savez_compressed(os.path.join(HERE, "imexq_adr.npz"), **out)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def norms(a: np.ndarray) -> dict:
    return {"max": float(a.max()).hex(), "min": float(a.min()).hex(), "absmax": float(np.abs(a).max()).hex(),
            "sum": float(np.sum(a, dtype=np.float64)).hex()}


def full(names):
    """Full-size fixtures through the unmodified reference (oracle/_ref)."""
    if O.ref_lib() is None:
        raise SystemExit("oracle/_ref not available (it travels prebuilt; build it where /root/reference exists)")
    for name in names:
        make, schemes = FULL[name]
        t0 = time.time()
        spec = make()
        gen_s = time.time() - t0
        out = {"config": name, "grid": list(spec.problem.n[: spec.problem.ndim]), "species": spec.problem.nspecies,
               "M": spec.M, "n_sweeps": spec.n_sweeps, "dt": spec.dt, "n_steps": 1, "nu": 1,
               "phi0_sha256": sha(spec.phi0), "generated_by": "oracle/_ref (unmodified cisdc::integrate / "
               "cisdc::execute_pipelined) driving the oracle problem class",
               "host": {"node": platform.node(), "nproc": os.cpu_count(),
                        "oracle_threads": int(os.environ.get("CISDC_ORACLE_THREADS", "1"))},
               "phi0_seconds": gen_s, "runs": {}}
        for s in schemes:
            workers = min(os.cpu_count() or 1, 6) if s == 2 else 0
            o = api.IntegrateOptions(scheme=s, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps, nu=1,
                                     workers=workers)
            t0 = time.time()
            f, reps, incs = O.ref_integrate(spec.problem, spec.phi0, o)
            wall = time.time() - t0
            r = reps[0]
            out["runs"][str(s)] = {
                "scheme": ["misdc", "misdcq", "cisdcq"][s], "workers": workers, "seconds": wall,
                "final_sha256": sha(f), "final_norms": norms(f),
                "sweeps": r.sweeps, "diffusion": r.counters.diffusion, "reaction": r.counters.reaction,
                "newton_iterations": r.counters.newton_iterations, "mg_cycles": r.counters.mg_cycles,
                "increments": [float(x).hex() for x in incs[: r.sweeps]],
            }
            print(name, s, f"{wall:.1f} s", out["runs"][str(s)]["final_sha256"][:16], flush=True)
            del f
        path = os.path.join(HERE, f"full_{name}.json")
        with open(path, "w") as fh:
            json.dump(out, fh, indent=1)
        print("wrote", path, flush=True)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--full":
        full(sys.argv[2:] or ["c3", "c4"])
        return
    if O.ref_lib() is None:
        raise SystemExit("oracle/_ref not available: build it with make -C oracle ref (needs /root/reference)")
    if len(sys.argv) > 1 and sys.argv[1] == "--imexq":
        imexq_adr()
        return
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
    imexq_adr()
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
