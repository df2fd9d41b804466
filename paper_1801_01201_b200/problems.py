"""Problem descriptions and the seeded BASELINE configurations.

A ``ProblemDesc`` is the host-side description handed across the C-ABI (cisdc_problem_desc of
include/cisdc_gpu.h).  It owns every array the C struct points to (velocity tables, diffusivities,
the reaction network), so CPU oracle and GPU engine are fed the *same bits*.

Configurations (BASELINE.json ``configs``; underspecified items resolved as in SURVEY.md App. C and
recorded in DESIGN.md):

  C0  the reference's own 1-D Dirichlet PDE on [0,20] (reaction_diffusion.hpp:28-99), n_x = 200,
      a = 1, d = 2, r = 4 -- the gate run against the UNMODIFIED reference code.
  C1  1-D periodic, N = 256, u = 1, d = 0.02, R = -1000 phi, gaussian, M = 2, 4 sweeps, dt = 1e-3, 100 steps.
  C2  1-D periodic, N = 65536, u = 1, d = 0.005, R = 1e4 phi(1-phi)(phi-0.3), 8 random Fourier modes,
      M = 4, 8 sweeps, dt = 5e-4, 200 steps, Newton tol 1e-12.
  C3  2-D periodic 1024^2, 3 species A->B->C->A (1, 1e2, 1e4), D = (0.01, 0.005, 0.001), vortex,
      32 modes, M = 4, 6 sweeps, dt = 1e-3, 10 steps, multigrid.
  C4  2-D periodic 2048^2, 9 species, 12 random mass-action reactions, M = 4, 8 sweeps, dt = 1e-5,
      2 steps, Newton tol 1e-12, multigrid.  (dt: the undamped Newton of the reference (cap 50) diverges
      for this network at dt >= 5e-5 -- rate constants up to 1e6 -- so dt is lowered as SURVEY App. C
      prescribes; measured on the CPU oracle.)
  C5  3-D periodic 256^3, 9 species (same network generator and seed), u = (1, 0.5, 0.25), 64 modes,
      M = 6, 10 sweeps, dt = 1e-5 (same reason), 1 step, PMISDC (CISDCQ nu = 1), multigrid to 1e-10.

Every generator takes ``scale`` (grid cells per axis divided by ``scale``) so parity tests run the
same physics at sizes the CPU oracle finishes in seconds.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi


@dataclass
class ProblemDesc:
    kind: int = _abi.PROBLEM_PERIODIC_ADR
    ndim: int = 1
    n: tuple = (8, 1, 1)
    nspecies: int = 1
    h: tuple = (1.0, 1.0, 1.0)
    vel: dict = field(default_factory=dict)  # (a, b) -> 1-D table along axis b, component a
    diffusivity: Optional[np.ndarray] = None
    reaction_kind: int = _abi.REACTION_NONE
    lam: float = 0.0
    theta: float = 0.0
    reactants: Optional[np.ndarray] = None  # (R, 2) int32, -1 = none
    products: Optional[np.ndarray] = None
    rate_constants: Optional[np.ndarray] = None
    newton_tol: float = 1e-14
    newton_max_iter: int = 50
    diffusion_solver: int = _abi.DIFFUSION_DIRECT
    mg_tol: float = 1e-10
    mg_max_cycles: int = 100
    mg_pre: int = 2
    mg_post: int = 2
    mg_coarse_sweeps: int = 8
    mg_min_coarse: int = 4
    mg_omega: float = 0.8
    ref_a: float = 0.0
    ref_d: float = 0.0
    ref_r: float = 0.0
    coupled_tol: float = 1e-13     # periodic ADR coupled stage (cisdc_gpu.h); used when coupled_max_iter > 0
    coupled_max_iter: int = 0      # 0: no coupled solve (IMEXQ raises CapabilityError, like the reference PDE)
    name: str = ""

    @property
    def ncell(self) -> int:
        return int(np.prod(self.n[: self.ndim])) if self.kind == _abi.PROBLEM_PERIODIC_ADR else self.n[0]

    @property
    def dim(self) -> int:
        if self.kind == _abi.PROBLEM_LINEAR_SCALAR:
            return 1
        if self.kind == _abi.PROBLEM_REFERENCE_RD:
            return self.n[0]
        return self.ncell * self.nspecies

    def to_c(self) -> _abi.ProblemDescC:
        d = _abi.ProblemDescC()
        d.kind = self.kind
        d.ndim = self.ndim
        for a in range(3):
            d.n[a] = int(self.n[a])
            d.h[a] = float(self.h[a])
        d.nspecies = self.nspecies
        self._keep = []
        for (a, b), tab in self.vel.items():
            arr = np.ascontiguousarray(tab, dtype=np.float64)
            self._keep.append(arr)
            d.vel[a][b] = _abi.dptr(arr)
        if self.diffusivity is not None:
            arr = np.ascontiguousarray(self.diffusivity, dtype=np.float64)
            self._keep.append(arr)
            d.diffusivity = _abi.dptr(arr)
        d.reaction_kind = self.reaction_kind
        d.lam = self.lam
        d.theta = self.theta
        if self.reactants is not None:
            r = np.ascontiguousarray(self.reactants, dtype=np.int32).reshape(-1)
            p = np.ascontiguousarray(self.products, dtype=np.int32).reshape(-1)
            k = np.ascontiguousarray(self.rate_constants, dtype=np.float64)
            self._keep += [r, p, k]
            d.n_reactions = len(k)
            d.reactants = _abi.iptr(r)
            d.products = _abi.iptr(p)
            d.rate_constants = _abi.dptr(k)
        d.newton_tol = self.newton_tol
        d.newton_max_iter = self.newton_max_iter
        d.diffusion_solver = self.diffusion_solver
        d.mg_tol = self.mg_tol
        d.mg_max_cycles = self.mg_max_cycles
        d.mg_pre = self.mg_pre
        d.mg_post = self.mg_post
        d.mg_coarse_sweeps = self.mg_coarse_sweeps
        d.mg_min_coarse = self.mg_min_coarse
        d.mg_omega = self.mg_omega
        d.ref_a, d.ref_d, d.ref_r = self.ref_a, self.ref_d, self.ref_r
        d.coupled_tol = self.coupled_tol
        d.coupled_max_iter = self.coupled_max_iter
        return d


@dataclass
class RunSpec:
    """A configuration: problem, initial state and the integrate options of its run."""
    problem: ProblemDesc
    phi0: np.ndarray
    scheme: int
    M: int
    n_sweeps: int
    dt: float
    n_steps: int
    nu: int = 1
    convention: int = 0
    name: str = ""
    schemes: tuple = ()


# ----------------------------------------------------------------------------- generators

def centers(n: int) -> np.ndarray:
    h = 1.0 / n
    return (np.arange(n, dtype=np.float64) + 0.5) * h


def faces(n: int) -> np.ndarray:
    h = 1.0 / n
    return np.arange(1, n + 1, dtype=np.float64) * h


def vortex_tables(nx: int, ny: int) -> dict:
    """u = (sin 2pi x cos 2pi y, -cos 2pi x sin 2pi y), sampled at the faces, separable."""
    tp = 2.0 * math.pi
    return {
        (0, 0): np.sin(tp * faces(nx)), (0, 1): np.cos(tp * centers(ny)),
        (1, 0): -np.cos(tp * centers(nx)), (1, 1): np.sin(tp * faces(ny)),
    }


def constant_velocity_tables(u: tuple, n: tuple) -> dict:
    return {(a, a): np.full(n[a], float(u[a])) for a in range(len(u)) if u[a] != 0.0}


def random_fourier_field(rng: np.random.Generator, shape: tuple, n_modes: int, amp_std: float, kmax: int) -> np.ndarray:
    """sum_m a_m cos(2 pi k_m . x + phase_m) at cell centres x = (i + 1/2)/n; shape = (nx[, ny[, nz]]).

    Integer wave vectors (|k_d| <= kmax, k != 0) keep the field periodic.  Evaluated as one inverse
    FFT of the sparse spectrum (the cell-centre half-shift is a phase factor), so a 256^3 field costs
    one FFT instead of n_modes full-grid cosines."""
    ndim = len(shape)
    spec = np.zeros(shape, dtype=np.complex128)
    for _ in range(n_modes):
        while True:
            k = rng.integers(-kmax, kmax + 1, size=ndim)
            if np.any(k != 0):
                break
        a = rng.normal(0.0, amp_std)
        ph = rng.uniform(0.0, 2.0 * math.pi)
        shift = sum(math.pi * k[d] / shape[d] for d in range(ndim))
        spec[tuple(int(k[d]) % shape[d] for d in range(ndim))] += a * np.exp(1j * (ph + shift))
    return np.real(np.fft.ifftn(spec)) * float(np.prod(shape))


def to_layout(fields_xyz: list) -> np.ndarray:
    """species list of arrays indexed [x, y, z] -> flat species-major, x-fastest layout."""
    return np.concatenate([np.ascontiguousarray(f.T).reshape(-1) for f in fields_xyz])


def random_network(rng: np.random.Generator, S: int, R: int) -> tuple:
    reac = -np.ones((R, 2), dtype=np.int32)
    prod = -np.ones((R, 2), dtype=np.int32)
    k = np.zeros(R)
    for r in range(R):
        nr = int(rng.integers(1, 3))
        npd = int(rng.integers(1, 3))
        reac[r, :nr] = rng.integers(0, S, size=nr)
        prod[r, :npd] = rng.integers(0, S, size=npd)
        k[r] = 10.0 ** rng.uniform(0.0, 6.0)
    return reac, prod, k


def mg_defaults(p: ProblemDesc, tol: float = 1e-10) -> ProblemDesc:
    p.diffusion_solver = _abi.DIFFUSION_MULTIGRID
    p.mg_tol = tol
    p.mg_max_cycles = 100
    p.mg_pre, p.mg_post, p.mg_coarse_sweeps, p.mg_min_coarse, p.mg_omega = 2, 2, 8, 4, 0.8
    return p


# ----------------------------------------------------------------------------- configs

def config_c0(n_x: int = 200, a: float = 1.0, d: float = 2.0, r: float = 4.0, dt: float = 0.05,
              n_steps: int = 20, M: int = 4, n_sweeps: int = 4) -> RunSpec:
    p = ProblemDesc(kind=_abi.PROBLEM_REFERENCE_RD, ndim=1, n=(n_x, 1, 1), nspecies=1,
                    ref_a=a, ref_d=d, ref_r=r, name="c0-reference-rd")
    dx = 20.0 / n_x
    x = (np.arange(n_x) + 0.5) * dx
    # initial_condition, reaction_diffusion.cpp:69-74 (libm tanh, like std::tanh)
    phi0 = np.array([0.5 * (1.0 + math.tanh(20.0 - 2.0 * float(xi))) for xi in x])
    return RunSpec(p, phi0, 1, M, n_sweeps, dt, n_steps, name="c0", schemes=(0, 1, 2))


def config_c1(scale: int = 1) -> RunSpec:
    N = 256 // scale
    p = ProblemDesc(ndim=1, n=(N, 1, 1), nspecies=1, h=(1.0 / N, 1, 1),
                    vel=constant_velocity_tables((1.0,), (N,)), diffusivity=np.array([0.02]),
                    reaction_kind=_abi.REACTION_LINEAR_DECAY, lam=1000.0, name="c1")
    x = centers(N)
    phi0 = np.exp(-((x - 0.5) ** 2) / 0.01)
    return RunSpec(p, phi0, 2, 2, 4, 1e-3, 100, nu=1, name="c1", schemes=(0, 2))


def config_c2(scale: int = 1, seed: int = 2, n_steps: int = 200) -> RunSpec:
    N = 65536 // scale
    p = ProblemDesc(ndim=1, n=(N, 1, 1), nspecies=1, h=(1.0 / N, 1, 1),
                    vel=constant_velocity_tables((1.0,), (N,)), diffusivity=np.array([0.005]),
                    reaction_kind=_abi.REACTION_BISTABLE, lam=1e4, theta=0.3, newton_tol=1e-12, name="c2")
    rng = np.random.default_rng(seed)
    x = centers(N)
    s = np.zeros(N)
    for _ in range(8):
        amp = rng.uniform(-1.0, 1.0)
        k = int(rng.integers(1, 17))
        ph = rng.uniform(0.0, 2.0 * math.pi)
        s += amp * np.sin(2.0 * math.pi * k * x + ph)
    phi0 = np.clip(0.5 + 0.5 * np.tanh(s), 0.0, 1.0)
    return RunSpec(p, phi0, 1, 4, 8, 5e-4, n_steps, name="c2", schemes=(0, 1, 2))


def config_c3(scale: int = 1, seed: int = 3, n_steps: int = 10) -> RunSpec:
    N = 1024 // scale
    p = ProblemDesc(ndim=2, n=(N, N, 1), nspecies=3, h=(1.0 / N, 1.0 / N, 1.0),
                    vel=vortex_tables(N, N), diffusivity=np.array([0.01, 0.005, 0.001]),
                    reaction_kind=_abi.REACTION_MASS_ACTION,
                    reactants=np.array([[0, -1], [1, -1], [2, -1]], dtype=np.int32),
                    products=np.array([[1, -1], [2, -1], [0, -1]], dtype=np.int32),
                    rate_constants=np.array([1.0, 1e2, 1e4]), name="c3")
    mg_defaults(p)
    p.mg_coarse_sweeps = 4  # more coarse-level sweeps do not reduce the V-cycle count (tools/mg_tune.py)
    rng = np.random.default_rng(seed)
    fields = [np.maximum(1.0 / 3.0 + random_fourier_field(rng, (N, N), 32, 0.1, 4), 1e-8) for _ in range(3)]
    return RunSpec(p, to_layout(fields), 1, 4, 6, 1e-3, n_steps, name="c3", schemes=(0, 1, 2))


def _c45_network(seed: int = 45):
    rng = np.random.default_rng(seed)
    reac, prod, k = random_network(rng, 9, 12)
    D = 10.0 ** rng.uniform(-4.0, -2.0, size=9)
    return reac, prod, k, D


def _normalised_fields(rng, shape, S, modes, kmax):
    f = [np.maximum(1.0 / S + random_fourier_field(rng, shape, modes, 0.1 / S, kmax), 1e-8) for _ in range(S)]
    tot = sum(f)
    return [x / tot for x in f]


def config_c4(scale: int = 1, seed: int = 4, n_steps: int = 2) -> RunSpec:
    N = 2048 // scale
    reac, prod, k, D = _c45_network()
    p = ProblemDesc(ndim=2, n=(N, N, 1), nspecies=9, h=(1.0 / N, 1.0 / N, 1.0), vel=vortex_tables(N, N),
                    diffusivity=D, reaction_kind=_abi.REACTION_MASS_ACTION, reactants=reac, products=prod,
                    rate_constants=k, newton_tol=1e-12, name="c4")
    mg_defaults(p)
    p.mg_coarse_sweeps = 2  # two levels here: 2 coarse sweeps already give the V-cycle count of 8
    rng = np.random.default_rng(seed)
    fields = _normalised_fields(rng, (N, N), 9, 32, 4)
    return RunSpec(p, to_layout(fields), 1, 4, 8, 1e-5, n_steps, name="c4", schemes=(0, 1, 2))


def config_c5(scale: int = 1, seed: int = 5, n_steps: int = 1) -> RunSpec:
    N = 256 // scale
    reac, prod, k, D = _c45_network()
    p = ProblemDesc(ndim=3, n=(N, N, N), nspecies=9, h=(1.0 / N,) * 3,
                    vel=constant_velocity_tables((1.0, 0.5, 0.25), (N, N, N)), diffusivity=D,
                    reaction_kind=_abi.REACTION_MASS_ACTION, reactants=reac, products=prod, rate_constants=k,
                    name="c5")
    mg_defaults(p, 1e-10)
    rng = np.random.default_rng(seed)
    fields = _normalised_fields(rng, (N, N, N), 9, 64, 4)
    return RunSpec(p, to_layout(fields), 2, 6, 10, 1e-5, n_steps, nu=1, name="c5", schemes=(2,))


CONFIGS = {"c0": config_c0, "c1": config_c1, "c2": config_c2, "c3": config_c3, "c4": config_c4, "c5": config_c5}


def linear_scalar(a: float, d: float, r: float, batch: int = 1) -> ProblemDesc:
    """LinearScalarProblem (proj/core/include/cisdc/problems/linear.hpp:31-51): phi' = (a + d + r) phi
    with exact stage solves and the coupled solve IMEXQ needs; `batch` independent copies (one per
    element, batch = 1 is the reference's dimension-1 problem)."""
    return ProblemDesc(kind=_abi.PROBLEM_LINEAR_SCALAR, ndim=1, n=(batch, 1, 1), ref_a=a, ref_d=d, ref_r=r,
                       name="linear")
