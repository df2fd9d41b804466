"""Multigrid parameter sweep on one config (dev helper, GPU): step time and V-cycles per step for
(pre, post, coarse) sweep counts.  The parameters are problem data, so the oracle follows the same
cycles (parity is unaffected); this only picks the defaults.

  python tools/mg_tune.py --config c4 --sets 2,2,8 2,2,4 4,4,8
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1801_01201_b200 import api, problems  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--scale", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--sets", nargs="+", default=["2,2,8"])
    a = ap.parse_args()
    for st in a.sets:
        pre, post, coarse = (int(v) for v in st.split(","))
        spec = problems.CONFIGS[a.config](scale=a.scale)
        spec.problem.mg_pre, spec.problem.mg_post, spec.problem.mg_coarse_sweeps = pre, post, coarse
        opt = api.IntegrateOptions(scheme=spec.scheme, dt=spec.dt, n_steps=1, M=spec.M, n_sweeps=spec.n_sweeps,
                                   nu=spec.nu, workers=2 if spec.scheme == 2 else 0)
        ctx = api.GpuContext(spec.problem, spec.M)
        api.integrate(spec.problem, spec.phi0, opt, ctx=ctx)  # warm-up (graphs, predictions)
        t0 = time.perf_counter()
        cyc = 0
        for _ in range(a.steps):
            r = api.integrate(spec.problem, spec.phi0, opt, ctx=ctx)
            cyc += r.steps[0].counters.mg_cycles
        dt = (time.perf_counter() - t0) / a.steps
        print(f"{a.config} pre={pre} post={post} coarse={coarse}: {dt * 1e3:.2f} ms/step, "
              f"{cyc / a.steps:.0f} species-cycles/step", flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
