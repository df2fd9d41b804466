"""Algorithmic work models for the roofline numbers bench.py reports.

Bytes: every kernel launch is charged its compulsory traffic (each distinct field read once and
written once; halo re-reads and constants are free) by the native library itself
(cisdc_gpu_kernel_times).  Flops: the batched Newton/LU kernel is FP64-bound for S = 9; its work is
counted analytically per Newton trip from the reaction network, as the specialised kernel executes
it: the static-pattern LU touches only the structurally non-zero entries of I - coef J and their
fill (csrc/rtc.cuh), so the count uses that pattern, not a dense S^3/3 (no pivot
comparisons or index arithmetic counted).
"""
from __future__ import annotations

import numpy as np

from . import _abi


def _network(desc):
    S = desc.nspecies
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
    return S, reac, nu


def lu_pattern(desc) -> np.ndarray:
    """Structural pattern of the LU factors of I - coef J (no row interchanges)."""
    S, reac, nu = _network(desc)
    pat = np.eye(S, dtype=bool)
    for r in range(len(reac)):
        for t in range(2):
            q = reac[r, t]
            if q >= 0:
                pat[nu[:, r] != 0, q] = True
    for k in range(S):
        rows = [i for i in range(k + 1, S) if pat[i, k]]
        cols = [j for j in range(k + 1, S) if pat[k, j]]
        for i in rows:
            pat[i, cols] = True
    return pat


def newton_flops(desc, sparse: bool = True) -> tuple[float, float]:
    """(flops of a residual-only trip, extra flops of a trip that builds and solves the Jacobian)."""
    if desc.reaction_kind != _abi.REACTION_MASS_ACTION:
        if desc.reaction_kind == _abi.REACTION_BISTABLE:
            return 7.0, 11.0  # f: 4 mul + 3 add/sub ; f': 7 ops + step/update/test 4
        return 4.0, 6.0
    S, reac, nu = _network(desc)
    nr = len(reac)
    rates = sum(2 if reac[r, 1] >= 0 else 1 for r in range(nr))
    residual = rates + 2 * int(np.count_nonzero(nu)) + 3 * S
    jac = 0
    jnz = np.zeros((S, S), dtype=bool)
    for r in range(nr):
        if not np.any(nu[:, r]):
            continue
        two = reac[r, 1] >= 0
        for t in range(2):
            q = reac[r, t]
            if q < 0:
                continue
            jac += 1 if two else 0  # g = k * x
            jac += 2 * int(np.count_nonzero(nu[:, r]))
            jnz[nu[:, r] != 0, q] = True
    if sparse:
        pat = lu_pattern(desc)
        shift = 2 * int(np.count_nonzero(jnz))
        lu = 0
        for k in range(S):
            cols = int(np.count_nonzero(pat[k, k + 1:]))
            for i in range(k + 1, S):
                if pat[i, k]:
                    lu += 1 + 2 * cols + 2  # m, row update, f update
        back = sum(2 * int(np.count_nonzero(pat[i, i + 1:])) + 1 for i in range(S))
    else:
        shift = 2 * S * S
        lu = sum((S - 1 - k) * (1 + 2 * (S - 1 - k) + 2) for k in range(S))
        back = sum(2 * (S - 1 - i) + 1 for i in range(S))
    update = S
    return float(residual), float(jac + shift + lu + back + update)


def rates_flops(desc) -> float:
    """FP64 flops of one F_R evaluation at a cell (the rates and the stoichiometric sums), the work
    the reaction kernel does after the solve for the stage's F_R output (eval_reaction)."""
    if desc.reaction_kind != _abi.REACTION_MASS_ACTION:
        return 4.0 if desc.reaction_kind == _abi.REACTION_BISTABLE else 1.0
    S, reac, nu = _network(desc)
    return float(sum(2 if reac[r, 1] >= 0 else 1 for r in range(len(reac))) + 2 * int(np.count_nonzero(nu)))


def newton_work(desc, trips: int, full_trips: int, sparse: bool = True, cell_solves: int = 0) -> float:
    """Lower-bound FP64 flops of `trips` Newton trips, `full_trips` of which built and solved the
    Jacobian (the others ended at the residual test |f| <= tol; the device counts those exits,
    cisdc_gpu_newton_residual_exits), plus the F_R evaluation at each of `cell_solves` results.
    Every trip evaluates the residual."""
    res, full = newton_flops(desc, sparse)
    return trips * res + max(full_trips, 0) * full + cell_solves * rates_flops(desc)
