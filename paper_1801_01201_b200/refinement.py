"""Temporal-order study on the GPU (refinement_study, proj/core/src/problems/refinement.cpp:26-122).

Errors are L1-mean distances (l1_error, reaction_diffusion.cpp:185-190) to a fine-step MISDCQ
reference at the same grid spacing (reference dt defaults to dx/32); slopes are least-squares fits of
log(err) against log(dt) (fit_loglog_slope, refinement.cpp:58-72).  Every integration runs on the GPU
through the C-ABI.  The reference's on-disk reference cache (SDC1 snapshots) is not used.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import api, problems


@dataclass
class RefinementOptions:  # refinement.hpp:29-42
    n_x: int = 200
    a: float = 1.0
    d: float = 2.0
    r: float = 4.0
    final_time: float = 0.4
    dt_list: tuple = (0.05, 0.025, 0.0125, 0.00625)
    sweep_counts: tuple = (2, 4, 8)
    schemes: tuple = (api.Scheme.misdc, api.Scheme.misdcq, api.Scheme.cisdcq)
    nu: int = 1
    M: int = 4
    convention: int = api.EulerConvention.cumulative
    ref_dt: float = 0.0
    ref_sweeps: int = 8


@dataclass
class RefinementCurve:
    scheme: int
    sweeps: int
    errors: list = field(default_factory=list)
    slope: float = 0.0
    slope_valid: bool = False


@dataclass
class RefinementResult:
    dt_list: tuple
    curves: list
    reference: np.ndarray


def steps_for(final_time: float, dt: float) -> int:
    n = int(round(final_time / dt))
    if n < 1 or abs(n * dt - final_time) > 1e-9 * final_time:
        raise ValueError("refinement_study: dt must divide the final time")
    return n


def fit_loglog_slope(dts, errors) -> float:
    if len(dts) != len(errors) or len(dts) < 2:
        raise ValueError("fit_loglog_slope: need at least two points")
    sx = sy = sxx = sxy = 0.0
    n = float(len(dts))
    for dt, e in zip(dts, errors):
        x, y = math.log(dt), math.log(e)
        sx += x
        sy += y
        sxx += x * x
        sxy += x * y
    return (n * sxy - sx * sy) / (n * sxx - sx * sx)


def refinement_study(opt: RefinementOptions, integrate=api.integrate) -> RefinementResult:
    if not opt.dt_list:
        raise ValueError("refinement_study: empty dt list")
    spec = problems.config_c0(n_x=opt.n_x, a=opt.a, d=opt.d, r=opt.r)
    dx = 20.0 / opt.n_x
    ref_dt = opt.ref_dt if opt.ref_dt > 0.0 else dx / 32.0

    def run(scheme, dt, sweeps, nu):
        o = api.IntegrateOptions(scheme=scheme, dt=dt, n_steps=steps_for(opt.final_time, dt), M=opt.M,
                                 n_sweeps=sweeps, nu=nu, convention=opt.convention)
        res = integrate(spec.problem, spec.phi0, o)
        return res.final_state if hasattr(res, "final_state") else res[0]

    reference = run(api.Scheme.misdcq, ref_dt, opt.ref_sweeps, 1)
    curves = []
    for scheme in opt.schemes:
        for sweeps in opt.sweep_counts:
            c = RefinementCurve(int(scheme), sweeps)
            for dt in opt.dt_list:
                sol = run(scheme, dt, sweeps, opt.nu)
                c.errors.append(float(np.mean(np.abs(sol - reference))))
            if len(opt.dt_list) >= 2:
                c.slope = fit_loglog_slope(opt.dt_list, c.errors)
                c.slope_valid = True
            curves.append(c)
    return RefinementResult(tuple(opt.dt_list), curves, reference)
