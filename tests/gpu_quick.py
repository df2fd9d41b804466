"""Quick GPU-vs-oracle parity sweep over all configs at reduced size (developer script)."""
import sys, os, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O
from paper_1801_01201_b200 import problems as P, api

def run(spec, scheme, nu=1, workers=0, steps=None, conv=0):
    steps = steps or spec.n_steps
    opt = api.IntegrateOptions(scheme=scheme, dt=spec.dt, n_steps=steps, M=spec.M, n_sweeps=spec.n_sweeps, nu=nu,
                               workers=workers, convention=conv)
    t = time.time(); res = api.integrate(spec.problem, spec.phi0, opt); tg = time.time() - t
    t = time.time(); ref, reps, incs = O.integrate(spec.problem, spec.phi0, opt); tc = time.time() - t
    err = np.max(np.abs(res.final_state - ref)) / max(np.max(np.abs(ref)), 1e-300)
    nt_g = sum(s.counters.newton_iterations for s in res.steps)
    nt_c = sum(r.counters.newton_iterations for r in reps)
    mg_g = sum(s.counters.mg_cycles for s in res.steps)
    mg_c = sum(r.counters.mg_cycles for r in reps)
    bit = np.array_equal(res.final_state, ref)
    print(f"{spec.name:4s} n={spec.problem.dim:8d} scheme={scheme} nu={nu} w={workers} steps={steps} relerr={err:.2e} bitwise={bit} "
          f"newton {nt_g}/{nt_c} mg {mg_g}/{mg_c} gpu {tg:.2f}s cpu {tc:.2f}s", flush=True)
    return err, nt_g == nt_c

ok = True
specs = [P.config_c0(n_steps=5), P.config_c1(), P.config_c2(scale=16, n_steps=5), P.config_c3(scale=16, n_steps=1),
         P.config_c4(scale=32, n_steps=1), P.config_c5(scale=16)]
for spec in specs:
    for scheme in (0, 1, 2):
        try:
            e, nm = run(spec, scheme)
            ok &= e <= 1e-10
        except Exception as ex:
            print(spec.name, scheme, "EXC", type(ex).__name__, ex, flush=True); ok = False
    try:
        e, nm = run(spec, 2, nu=2, workers=2)
        ok &= e <= 1e-10
    except Exception as ex:
        print(spec.name, "pipelined EXC", type(ex).__name__, ex, flush=True); ok = False
print("ALL OK" if ok else "FAILURES")
