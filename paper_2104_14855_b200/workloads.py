"""Workload definitions and seeded synthetic inputs.

This module holds NONE of the method's arithmetic: it only names the five
configurations of BASELINE.json and draws the seeded inputs that both the
product path and the oracle consume (reading R-seed):

  * potential of the advecting field at the finest-level vertices (BASELINE.json):
      2D: stream function psi with vcurl psi = (sin^2(pi x) sin(2 pi y), -sin(2 pi x) sin^2(pi y))
      3D: vector potential A = sum_{k=1..3} a_k sin(k pi x) sin(k pi y) sin(k pi z) e_k,
          a_k ~ N(0,1) from the seed; the field is curl A
  * right-hand side b ~ U(-1,1) (n values), then an initial guess x0 ~ U(-1,1).

Draw order from numpy Generator(PCG64(seed)): a_1..a_3 (3D only), b, x0.
The paper's own workloads (lid-driven cavity, island coalescence; PAPER.md
P:683) need its nonlinear solver and k=2 elements; these synthetic
inputs stand in for them with the shapes of BASELINE.json.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    block: str          # "eb" (E-B block) or "vel" (AL velocity block)
    dim: int
    N: int              # finest cells per side
    levels: int
    Re: float
    Rem: float
    S: float
    gamma: float
    nu: int             # pre = post smoothing sweeps per level (reading R-nu)
    sigma: float = 10.0  # SIPG penalty 10 k^2, k = 1
    mu: float = 0.0      # Burman stabilisation (off, reading R-mu)
    theta: float = 1.0
    dt: float = 0.0      # NEXT-4: > 0 -> transient, (1/dt) mass terms
    picard: int = 0      # NEXT-4: 1 -> Picard linearisation, delta = 0
    degree: int = 1      # NEXT-2: element degree k; k = 2 for the 2D E-B block (CG2 x RT2)
    weights_mode: int = 0  # update weights w_i: 0 by degree, 1 per-DoF 1/m_d, 2 uniform 1/max m_d
    newton_reaction: int = 0  # (u . grad u^n, v) of Table 1 row F: zero under R-w (reading R-newton)

    @property
    def block_id(self) -> int:
        return 0 if self.block == "eb" else 1


CONFIGS = {
    # BASELINE.json configs[0..4]
    "c1": Config("c1", "eb", 2, 8, 2, Re=1.0, Rem=1.0, S=1.0, gamma=1.0, nu=1),
    "c2": Config("c2", "eb", 2, 128, 5, Re=1.0, Rem=1e3, S=1e3, gamma=1.0, nu=2),
    "c3": Config("c3", "vel", 2, 256, 6, Re=1e4, Rem=1.0, S=1.0, gamma=1e4, nu=2),
    "c4": Config("c4", "eb", 3, 32, 4, Re=1.0, Rem=1e3, S=1e3, gamma=1.0, nu=2),
    "c5": Config("c5", "vel", 3, 48, 4, Re=1e4, Rem=1.0, S=1.0, gamma=1e4, nu=2),
}


def small(name: str, N: int, levels: int) -> Config:
    """A reduced-size variant of a configuration (same block and parameters)."""
    return dataclasses.replace(CONFIGS[name], name=f"{name}-N{N}L{levels}", N=N, levels=levels)


def vertex_coords(dim: int, N: int) -> np.ndarray:
    """Finest-level vertex coordinates in vertex-id order i + (N+1)(j + (N+1)k)."""
    g = np.arange(N + 1, dtype=np.float64) / N
    if dim == 2:
        y, x = np.meshgrid(g, g, indexing="ij")
        return np.stack([x.ravel(), y.ravel()], axis=1)
    z, y, x = np.meshgrid(g, g, g, indexing="ij")
    return np.stack([x.ravel(), y.ravel(), z.ravel()], axis=1)


def advecting_potential(cfg: Config, a: np.ndarray | None) -> np.ndarray:
    """Potential of the advecting field at the finest vertices (reading R-w).

    2D: stream function psi = sin^2(pi x) sin^2(pi y) / pi, so that vcurl psi =
        (d_y psi, -d_x psi) = (sin^2(pi x) sin(2 pi y), -sin(2 pi x) sin^2(pi y)),
        the field of BASELINE.json configs 1-3 (1 value per vertex).
    3D: vector potential A = sum_k a_k sin(k pi x) sin(k pi y) sin(k pi z) e_k of
        BASELINE.json configs 4-5 (3 values per vertex); the field is u = curl A.
    """
    X = vertex_coords(cfg.dim, cfg.N)
    pi = math.pi
    if cfg.dim == 2:
        x, y = X[:, 0], X[:, 1]
        return np.ascontiguousarray(np.sin(pi * x) ** 2 * np.sin(pi * y) ** 2 / pi)
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    A = np.zeros((X.shape[0], 3))
    for k in (1, 2, 3):
        A[:, k - 1] = a[k - 1] * np.sin(k * pi * x) * np.sin(k * pi * y) * np.sin(k * pi * z)
    return np.ascontiguousarray(A.ravel())


def draw(cfg: Config, n: int, seed: int):
    """(potential, b, x0) for a configuration with n free finest-level DoFs."""
    rng = np.random.Generator(np.random.PCG64(seed))
    a = rng.standard_normal(3) if cfg.dim == 3 else None
    w = advecting_potential(cfg, a)
    b = rng.uniform(-1.0, 1.0, n)
    x0 = rng.uniform(-1.0, 1.0, n)
    return w, b, x0


def magnetic_potential(cfg: Config, seed: int) -> np.ndarray:
    """Potential of a synthetic magnetic field B^n at the finest vertices (NEXT-4, the
    Lorentz term S(B^n x (u x B^n), v) of the velocity block).  Drawn from its own
    stream Generator(PCG64(seed + 7919)) so that the draws of draw() are unchanged:
      2D: phi = sum_{k=1,2} c_k sin(k pi x) sin(k pi y), B^n = vcurl phi_h;
      3D: A = sum_{k=1..3} c_k sin(k pi x) sin(k pi y) sin(k pi z) e_k, B^n = curl A_h;
    c_k ~ N(0,1).  B^n . n = 0 on the boundary, as the paper's B."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    X = vertex_coords(cfg.dim, cfg.N)
    pi = math.pi
    if cfg.dim == 2:
        c = rng.standard_normal(2)
        x, y = X[:, 0], X[:, 1]
        return np.ascontiguousarray(sum(c[k - 1] * np.sin(k * pi * x) * np.sin(k * pi * y) for k in (1, 2)))
    c = rng.standard_normal(3)
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    A = np.zeros((X.shape[0], 3))
    for k in (1, 2, 3):
        A[:, k - 1] = c[k - 1] * np.sin(k * pi * x) * np.sin(k * pi * y) * np.sin(k * pi * z)
    return np.ascontiguousarray(A.ravel())
