"""Problem definitions, BASELINE configs and seeded synthetic inputs.

Two groups:
* the reference's own 1D FEM problems (heat / monodomain), mirroring
  paradiff/problems.py:1-112;
* the BASELINE.json configs C1..C5 (Dirichlet/periodic finite differences in
  1-3D, Fisher or cubic reaction), which the reference only runs through
  injected operators.  Scaling is FEM-consistent:
  Kh = coef * h^d * (-Lap_h), Mh = h^d * I, so tolerances on unscaled
  residual norms behave like the reference's FEM path.

All inputs are generated on the host in fp64 with numpy.random.default_rng
(seed) — there is no public dataset; SURVEY §8(d) fixes the recipes.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np
import scipy.sparse as sp

from .errors import ConfigurationError
from .fem1d import SpaceMesh, SpaceOperators, semidiscrete_rates


# ------------------------------------------------------------------ stencils
@dataclass(frozen=True)
class StencilSpec:
    """Structured description of a spatial operator Kh = coef*h^d*(-Lap_h).

    bc: "dirichlet" (n interior points per axis, h = 1/(n+1)) or "periodic"
    (n points per axis, h = 1/n).  Flat index is C-order over the axes, the
    last axis fastest, matching kron(T, I) + kron(I, T).
    """

    dim: int
    n: int
    bc: str
    coef: float = 1.0

    @property
    def h(self) -> float:
        return 1.0 / (self.n + 1) if self.bc == "dirichlet" else 1.0 / self.n

    @property
    def ndof(self) -> int:
        return self.n ** self.dim

    @property
    def mass(self) -> float:
        return self.h ** self.dim

    def coarse(self) -> "StencilSpec":
        if self.bc == "dirichlet":
            if self.n % 2 == 0 or self.n < 3:
                raise ConfigurationError(f"cannot coarsen {self.n} Dirichlet interior points")
            return StencilSpec(self.dim, (self.n - 1) // 2, self.bc, self.coef)
        if self.n % 2 or self.n < 4:
            raise ConfigurationError(f"cannot coarsen {self.n} periodic points")
        return StencilSpec(self.dim, self.n // 2, self.bc, self.coef)


def _second_difference(n: int, bc: str) -> sp.csr_matrix:
    T = sp.diags([np.full(n - 1, -1.0), np.full(n, 2.0), np.full(n - 1, -1.0)], [-1, 0, 1],
                 format="lil")
    if bc == "periodic":
        T[0, n - 1] += -1.0
        T[n - 1, 0] += -1.0
    elif bc != "dirichlet":
        raise ConfigurationError(f"unknown boundary condition {bc!r}")
    return sp.csr_matrix(T)


def _kron_sum(T: sp.csr_matrix, dim: int) -> sp.csr_matrix:
    n = T.shape[0]
    eye = sp.eye(n, format="csr")
    out = None
    for axis in range(dim):
        term = None
        for a in range(dim):
            f = T if a == axis else eye
            term = f if term is None else sp.kron(term, f, format="csr")
        out = term if out is None else out + term
    return out


def stencil_matrix(spec: StencilSpec) -> sp.csr_matrix:
    h = spec.h
    lap = _kron_sum(_second_difference(spec.n, spec.bc), spec.dim) / h**2
    K = sp.csr_matrix(spec.coef * h**spec.dim * lap)
    K.sum_duplicates()
    K.sort_indices()
    return K


def fd_space(spec: StencilSpec) -> SpaceOperators:
    """SpaceOperators for a structured FD operator (mesh.ndof == spec.ndof)."""
    S = spec.ndof
    Kh = stencil_matrix(spec)
    Mh = sp.diags(np.full(S, spec.mass), format="dia")
    return SpaceOperators(mesh=SpaceMesh(S - 1, 1.0), Kh=Kh, Mh=Mh,
                          MhConsistent=sp.csr_matrix(Mh), stencil=spec)


def _restriction_1d(n: int, bc: str) -> sp.csr_matrix:
    if bc == "dirichlet":
        nc = (n - 1) // 2
        R = sp.lil_matrix((nc, n))
        for i in range(nc):
            R[i, 2 * i], R[i, 2 * i + 1], R[i, 2 * i + 2] = 0.25, 0.5, 0.25
    else:
        nc = n // 2
        R = sp.lil_matrix((nc, n))
        for i in range(nc):
            R[i, (2 * i - 1) % n] += 0.25
            R[i, 2 * i] += 0.5
            R[i, 2 * i + 1] += 0.25
    return sp.csr_matrix(R)


def fd_transfers(spec: StencilSpec) -> tuple[sp.csr_matrix, sp.csr_matrix]:
    """Full weighting R (tensor [1,2,1]/4) and P = 2^d R^T (bi/trilinear)."""
    spec.coarse()
    R1 = _restriction_1d(spec.n, spec.bc)
    R = R1
    for _ in range(spec.dim - 1):
        R = sp.kron(R, R1, format="csr")
    R = sp.csr_matrix(R)
    R.sort_indices()
    P = sp.csr_matrix((2.0 ** spec.dim) * R.T)
    P.sort_indices()
    return R, P


def fd_grid(spec: StencilSpec) -> list[np.ndarray]:
    h = spec.h
    if spec.bc == "dirichlet":
        x = h * np.arange(1, spec.n + 1)
    else:
        x = h * np.arange(spec.n)
    return np.meshgrid(*([x] * spec.dim), indexing="ij")


# ------------------------------------------------------------------ reference problems
@dataclass(frozen=True)
class ProblemSpec:
    name: str
    X: float
    T: float
    gamma: float
    u0: Callable[[np.ndarray], np.ndarray]
    exact: Callable[[np.ndarray, float], np.ndarray] | None = None

    def __post_init__(self):
        if self.X <= 0 or self.T <= 0:
            raise ConfigurationError("domain length and final time must be positive")
        if self.gamma < 0:
            raise ConfigurationError("reaction intensity must be nonnegative")


_HEAT_MODES = ((1, 1.0), (3, 2.0), (4, 3.0))


def heat_problem() -> ProblemSpec:
    def u0(x):
        x = np.asarray(x, dtype=float)
        return sum(a * np.cos(k * np.pi * x) for k, a in _HEAT_MODES)

    def exact(x, t):
        x = np.asarray(x, dtype=float)
        return sum(a * np.cos(k * np.pi * x) * np.exp(-((k * np.pi) ** 2) * t)
                   for k, a in _HEAT_MODES)

    return ProblemSpec("heat", 1.0, 1.0, 0.0, u0, exact)


def heat_semidiscrete_exact(mesh: SpaceMesh):
    rates = {k: semidiscrete_rates(mesh, k) for k, _ in _HEAT_MODES}

    def exact(x, t):
        x = np.asarray(x, dtype=float)
        return sum(a * np.cos(k * np.pi * x) * np.exp(rates[k] * t) for k, a in _HEAT_MODES)

    return exact


def monodomain_problem() -> ProblemSpec:
    def u0(x):
        x = np.asarray(x, dtype=float)
        return 2.0 * np.exp(-(((x - 5.0) / 0.1) ** 2))

    return ProblemSpec("monodomain", 10.0, 2.0, 5.0, u0, None)


def get_problem(name: str) -> ProblemSpec:
    if name == "heat":
        return heat_problem()
    if name == "monodomain":
        return monodomain_problem()
    raise ConfigurationError(f"unknown problem {name!r}; expected 'heat' or 'monodomain'")


def error_norms(u_num, reference, system):
    """(max error at T, per-element end-node max errors); problems.py:92-106."""
    xs = system.space.mesh.vertices
    steps = system.as_steps(u_num)
    per = np.array([np.max(np.abs(steps[n, -1] - reference(xs, (n + 1) * system.grid.dt)))
                    for n in range(system.grid.Nt)])
    return float(per[-1]), per


def spatial_mean(space, values) -> float:
    w = space.lumped_diagonal
    return float(np.dot(w, values) / np.sum(w))


# ------------------------------------------------------------------ BASELINE configs
@dataclass(frozen=True)
class BaselineConfig:
    """One BASELINE.json config (possibly at a reduced, labelled size)."""

    name: str
    spec: StencilSpec
    Nt: int
    T: float
    M: int
    M_coarse: int
    gamma: float
    reaction: str     # "cubic" (u^3-u) or "fisher" (u^2-u)
    seed: int = 0
    reduced: str = ""

    @property
    def dt(self) -> float:
        return self.T / self.Nt

    @property
    def ndof(self) -> int:
        return self.Nt * self.M * self.spec.ndof

    def u0(self) -> np.ndarray:
        return config_u0(self)


def baseline_config(name: str, *, n: int | None = None, Nt: int | None = None,
                    seed: int = 0) -> BaselineConfig:
    """C1..C5 from BASELINE.json (full size unless n/Nt override, then labelled)."""
    table = {
        # name: (dim, n, bc, coef, Nt, T, M, Mc, gamma, reaction)
        "C1": (1, 127, "dirichlet", 0.1, 16, 1.0, 3, 2, 0.0, "cubic"),
        "C2": (2, 255, "dirichlet", 1.0, 64, 1.0, 3, 2, 0.0, "cubic"),
        "C3": (2, 512, "periodic", 1.0, 128, 1.28, 3, 2, 1.0, "fisher"),
        "C4": (3, 127, "dirichlet", 1.0, 256, 1.0, 5, 3, 0.0, "cubic"),
        "C5": (3, 256, "periodic", 0.1, 32, 0.032, 3, 2, 1.0, "cubic"),
    }
    if name not in table:
        raise ConfigurationError(f"unknown config {name!r}")
    dim, n0, bc, coef, nt0, T0, M, Mc, gamma, reaction = table[name]
    dt = T0 / nt0
    nn = n0 if n is None else n
    nt = nt0 if Nt is None else Nt
    reduced = "" if (nn == n0 and nt == nt0) else f"reduced from n={n0},Nt={nt0}"
    return BaselineConfig(name, StencilSpec(dim, nn, bc, coef), nt, dt * nt, M, Mc, gamma,
                          reaction, seed, reduced)


def config_u0(cfg: BaselineConfig) -> np.ndarray:
    """Seeded initial states, frozen recipes of SURVEY §8(d)."""
    rng = np.random.default_rng(cfg.seed)
    spec = cfg.spec
    grid = fd_grid(spec)
    if cfg.name in ("C1", "C2", "C4"):
        modes = {"C1": 5, "C2": 8, "C4": 16}[cfg.name]
        if spec.dim == 1:
            amps = rng.uniform(-1.0, 1.0, modes)
            u = sum(a * np.sin((k + 1) * np.pi * grid[0]) for k, a in enumerate(amps))
        else:
            ks = rng.integers(1, 9, size=(modes, spec.dim))
            amps = rng.uniform(-1.0, 1.0, modes)
            u = np.zeros_like(grid[0])
            for kv, a in zip(ks, amps):
                term = np.full_like(grid[0], a)
                for axis, k in enumerate(kv):
                    term = term * np.sin(k * np.pi * grid[axis])
                u = u + term
        return np.ascontiguousarray(u.ravel())
    if cfg.name == "C3":
        u = rng.uniform(0.0, 1.0, (spec.n,) * spec.dim)
        for _ in range(10):
            acc = np.zeros_like(u)
            for axis in range(spec.dim):
                acc += np.roll(u, 1, axis) + np.roll(u, -1, axis)
            u = acc / (2 * spec.dim)
        return np.ascontiguousarray(u.ravel())
    u = rng.uniform(-1.0, 1.0, (spec.n,) * spec.dim)
    return np.ascontiguousarray(u.ravel())
