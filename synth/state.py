"""Seeded simulation state and material inputs (no method arithmetic).

Recipes follow SURVEY.md §8(d) and DESIGN.md "Input recipe":
  * displacement ``u = X diag(sx, sy, sz) + U(-a/n, a/n)`` per component,
    zero on fixed vertices (so O8's "fixed vertices keep u = v = 0" holds);
  * fixed (Dirichlet) vertices: ``X_x <= min X_x + 0.5/n`` (SURVEY §8(c)
    reading for the paper's "same external conditions");
  * Lame parameters from Young's modulus and Poisson ratio (standard
    isotropic conversion; the paper only says "material properties on the
    tetrahedra") -- these are *inputs* to both sides.
"""
from __future__ import annotations

import numpy as np

from .mesh import rng


def fixed_mask(X: np.ndarray, n: int) -> np.ndarray:
    """uint8 per vertex, 1 = free, 0 = fixed (projection mask of O10)."""
    fixed = X[:, 0] <= X[:, 0].min() + 0.5 / n
    return (~fixed).astype(np.uint8)


def stretch_noise_u(X, n, seed, stretch=(0.1, -0.05, 0.0), noise=0.05, free=None, wall_ramp=0.0):
    """``wall_ramp = w > 0`` scales the stretch by clip((x - x_min) / w, 0, 1):
    the plain recipe pins the wall layer (u = 0) next to free vertices with
    u_y = -0.05 y, a shear of ~0.05 n that inverts tets beyond n ~ 200 (C5);
    the ramp keeps the shear at 0.05 / w for every n."""
    u = X * np.asarray(stretch, dtype=np.float64)[None, :]
    if wall_ramp > 0:
        u = u * np.clip((X[:, 0:1] - X[:, 0].min()) / wall_ramp, 0.0, 1.0)
    u = u + rng(seed).uniform(-noise / n, noise / n, size=X.shape)
    if free is not None:
        u[free == 0] = 0.0
    return u


def twist_u(X, n, seed, theta_per_z=0.3, stretch=1.1, noise=0.05, free=None):
    """C3 state: twist about the z axis through the domain centre + stretch."""
    c = np.array([0.5, 0.5, 0.5])
    d = X - c
    th = theta_per_z * X[:, 2]
    cs, sn = np.cos(th), np.sin(th)
    y = np.empty_like(X)
    y[:, 0] = c[0] + stretch * (cs * d[:, 0] - sn * d[:, 1])
    y[:, 1] = c[1] + stretch * (sn * d[:, 0] + cs * d[:, 1])
    y[:, 2] = c[2] + stretch * d[:, 2]
    u = y - X + rng(seed).uniform(-noise / n, noise / n, size=X.shape)
    if free is not None:
        u[free == 0] = 0.0
    return u


def lame(E, nu):
    E = np.asarray(E, dtype=np.float64)
    mu = E / (2.0 * (1.0 + nu))
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    return mu, lam


def materials(T: int, E: float, nu: float, spread: float = 0.0, seed: int = 5):
    """Per-tet (mu, lambda); ``spread`` = relative +-variation of E (C3: 0.1)."""
    Es = np.full(T, E, dtype=np.float64)
    if spread:
        Es = Es * (1.0 + rng(seed).uniform(-spread, spread, size=T))
    return lame(Es, nu)


# Named presets (BASELINE.json configs).
PRESETS = {
    # C1: StVK explicit, fp64, 10 steps, h = 1e-4, E = 1e6, nu = .3, rho = 1e3
    "C1": dict(mesh="kuhn6", n=4, model="stvk", E=1e6, nu=0.3, rho=1e3, h=1e-4, steps=10,
               u_seed=1, order_seed=None, dtype="f64"),
    # C2: NH implicit step + 50 PCG iterations, fp64, E = 2e5 so h^2 E n^2 / rho ~ 60
    "C2": dict(mesh="kuhn6", n=55, model="nh", E=2e5, nu=0.3, rho=1e3, h=1e-2, cg_iters=50,
               u_seed=1, order_seed=2, dtype="f64"),
    # C3: StVK force+stiffness map on a 1e7-tet blob, fp32
    "C3": dict(mesh="blob", T=10_000_000, model="stvk", E=1e6, nu=0.3, rho=1e3, spread=0.1,
               u_seed=6, dtype="f32"),
}
