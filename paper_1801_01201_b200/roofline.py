"""Algorithmic work models for the roofline numbers bench.py reports.

Bytes: every kernel launch is charged its compulsory traffic (each distinct field read once and
written once; halo re-reads and constants are free) by the native library itself
(cisdc_gpu_kernel_times).  Flops: the batched Newton/LU kernel is FP64-bound for S = 9; its work is
counted analytically per Newton trip from the reaction network (no pivot comparisons, no index
arithmetic), as SURVEY.md section 8(d) prescribes.
"""
from __future__ import annotations

import numpy as np

from . import _abi


def newton_flops(desc) -> tuple[float, float]:
    """(flops of a residual-only trip, extra flops of a trip that builds and solves the Jacobian)."""
    S = desc.nspecies
    if desc.reaction_kind != _abi.REACTION_MASS_ACTION:
        if desc.reaction_kind == _abi.REACTION_BISTABLE:
            return 7.0, 11.0  # f: 4 mul + 3 add/sub ; f': 7 ops + step/update/test 4
        return 4.0, 6.0
    reac = np.asarray(desc.reactants).reshape(-1, 2)
    prod = np.asarray(desc.products).reshape(-1, 2)
    nr = len(reac)
    nu = np.zeros((S, nr), dtype=int)
    for r in range(nr):
        for t in range(2):
            if reac[r, t] >= 0:
                nu[reac[r, t], r] -= 1
            if prod[r, t] >= 0:
                nu[prod[r, t], r] += 1
    nnz = int(np.count_nonzero(nu))
    rates = sum(2 if reac[r, 1] >= 0 else 1 for r in range(nr))
    residual = rates + 2 * nnz + 3 * S
    jac = 0
    for r in range(nr):
        nreac = 2 if reac[r, 1] >= 0 else 1
        jac += (1 if nreac == 2 else 0) + (1 if nreac == 2 else 0)  # g per reactant slot
        jac += 2 * int(np.count_nonzero(nu[:, r])) * nreac
    shift = 2 * S * S
    lu = sum((S - 1 - k) + 2 * (S - 1 - k) ** 2 for k in range(S))
    solves = sum(2 * i for i in range(S)) + sum(2 * (S - 1 - i) + 1 for i in range(S))
    update = S
    return float(residual), float(jac + shift + lu + solves + update)


def newton_work(desc, trips: int, cell_solves: int) -> float:
    """Lower-bound FP64 flops of `trips` Newton trips over `cell_solves` per-cell solves (each solve's
    last trip is counted as residual-only)."""
    res, full = newton_flops(desc)
    return trips * res + max(trips - cell_solves, 0) * full
