"""Shared test helpers: build the same seeded case for the oracle and the GPU."""
from __future__ import annotations

import numpy as np

import oracle
from synth import mesh as M
from synth import state as S


class Case:
    """Seeded workload in input order (SURVEY §8(d) recipe)."""

    def __init__(self, n=4, model="nh", E=2e5, nu=0.3, rho=1e3, mesh="kuhn6", order_seed=2, u_seed=1,
                 spread=0.0, vel_amp=0.0):
        if mesh == "kuhn6":
            X, tets = M.kuhn6(n)
        elif mesh == "alt5":
            X, tets = M.alt5(n)
        else:
            raise ValueError(mesh)
        if order_seed is not None:
            X, tets = M.permute_vertices(X, tets, order_seed)
            tets = M.permute_tets(tets, order_seed + 100)
        self.n, self.model, self.rho = n, model, rho
        self.X, self.tets = X, tets
        self.free = S.fixed_mask(X, n)
        self.u = S.stretch_noise_u(X, n, u_seed, free=self.free)
        self.vel = np.zeros_like(X)
        if vel_amp:
            self.vel = M.rng(u_seed + 7).uniform(-vel_amp, vel_amp, size=X.shape) * self.free[:, None]
        self.mu, self.lam = S.materials(tets.shape[0], E, nu, spread=spread)


def oracle_renumbered(case: Case):
    """Oracle O3 applied to the case, then the oracle mesh in the new order.

    Returns (mesh, new_of_old, tet_src) so that results can be compared row by
    row with the GPU's stored order (which must equal the oracle's O3 order).
    """
    new_of_old, tet_src, tets_new = oracle.renumber(case.X, case.tets)
    order = np.argsort(new_of_old)
    Xn = case.X[order]
    m = oracle.Mesh(Xn, tets_new, rho=case.rho)
    return m, new_of_old, tet_src, order


def gpu_fem(ctx, case: Case, dtype="f64", renumber=True, name="mesh", mass="lumped"):
    from paper_1506_07577_b200.tetfem import TetFEM
    return TetFEM(ctx, case.X, case.tets, dtype=dtype, mu=case.mu, lam=case.lam, rho=case.rho, free=case.free,
                  u=case.u, vel=case.vel, renumber=renumber, name=name, mass=mass)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d > 0 else 1.0))
