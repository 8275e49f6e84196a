"""Pins for oracle O6/O7 (element forces, stiffness, energy) and the edge matvec.

Independent checks only: rest state, translation/rotation invariance, finite
differences of the energy and of the forces, hand-derived closed forms for
homogeneous deformations, the linear-elastic limit W B^T D B (Voigt), the
patch test, and dense assembly by finite differences.
"""
import numpy as np
import pytest

import oracle
from synth import mesh as M
from synth import state as S

MODELS = ["stvk", "nh"]


def _mesh(gen=lambda: M.kuhn6(2)):
    X, tets = gen()
    return oracle.Mesh(X, tets)


def _rand_u(X, seed, amp=0.05):
    return np.random.default_rng(seed).uniform(-amp, amp, size=X.shape)


def _mat(m, mu=2.0, lam=3.0):
    return np.full(m.nt, mu), np.full(m.nt, lam)


def _f(model, m, u, mu, lam):
    return oracle.element_map(model, m.X, u, m.tets, m.Dminv, m.W, mu, lam, e=m.e, ne=m.ne)


@pytest.mark.parametrize("model", MODELS)
def test_rest_state_zero_force(model):
    m = _mesh()
    mu, lam = _mat(m)
    f, K, en, inv = _f(model, m, np.zeros_like(m.X), mu, lam)
    assert np.abs(f).max() < 1e-14 and abs(en) < 1e-15 and inv == 0


@pytest.mark.parametrize("model", MODELS)
def test_force_balance_and_torque(model):
    m = _mesh()
    mu, lam = _mat(m)
    u = _rand_u(m.X, 1)
    f, K, en, inv = _f(model, m, u, mu, lam)
    x = m.X + u
    scale = np.abs(f).max()
    assert np.abs(f.sum(axis=0)).max() < 1e-13 * scale * m.nv
    assert np.abs(np.cross(x, f).sum(axis=0)).max() < 1e-13 * scale * m.nv


@pytest.mark.parametrize("model", MODELS)
def test_force_is_minus_energy_gradient(model):
    m = _mesh(M.two_tets)
    mu, lam = _mat(m)
    u = _rand_u(m.X, 2, 0.1)
    f, _, _, _ = _f(model, m, u, mu, lam)
    eps = 1e-6
    g = np.zeros_like(u)
    for v in range(m.nv):
        for a in range(3):
            up, um = u.copy(), u.copy()
            up[v, a] += eps
            um[v, a] -= eps
            ep = _f(model, m, up, mu, lam)[2]
            em = _f(model, m, um, mu, lam)[2]
            g[v, a] = (ep - em) / (2 * eps)
    assert np.abs(f + g).max() < 1e-8 * max(1.0, np.abs(f).max())


def _dense(m, K):
    D = np.zeros((3 * m.nv, 3 * m.nv))
    for r in range(m.ne):
        a, b = m.tail[r], m.head[r]
        D[3 * a:3 * a + 3, 3 * b:3 * b + 3] = K[r]
    return D


@pytest.mark.parametrize("model", MODELS)
def test_stiffness_is_minus_force_jacobian(model):
    m = _mesh(M.two_tets)
    mu, lam = _mat(m)
    u = _rand_u(m.X, 3, 0.1)
    _, K, _, _ = _f(model, m, u, mu, lam)
    Kd = _dense(m, K)
    eps = 1e-6
    J = np.zeros_like(Kd)
    for v in range(m.nv):
        for a in range(3):
            up, um = u.copy(), u.copy()
            up[v, a] += eps
            um[v, a] -= eps
            J[:, 3 * v + a] = -(_f(model, m, up, mu, lam)[0] - _f(model, m, um, mu, lam)[0]).ravel() / (2 * eps)
    assert np.abs(Kd - J).max() < 1e-7 * np.abs(Kd).max()
    assert np.abs(Kd - Kd.T).max() < 1e-13 * np.abs(Kd).max()
    # translations are in the kernel
    for a in range(3):
        t = np.zeros((m.nv, 3))
        t[:, a] = 1.0
        assert np.abs(Kd @ t.ravel()).max() < 1e-12 * np.abs(Kd).max()


def test_linear_elastic_limit():
    """At F = I both models reduce to W B^T D B with the Voigt isotropic D."""
    m = _mesh(M.single_tet)
    mu, lam = 2.0, 3.0
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[:3, :3] += 2 * mu * np.eye(3)
    D[3:, 3:] = mu * np.eye(3)
    g = np.vstack([-m.Dminv[0].sum(axis=0), m.Dminv[0]])   # g_0 .. g_3 (rows of Dminv)
    B = np.zeros((6, 12))
    for i in range(4):
        gx, gy, gz = g[i]
        B[:, 3 * i:3 * i + 3] = [[gx, 0, 0], [0, gy, 0], [0, 0, gz], [gy, gx, 0], [0, gz, gy], [gz, 0, gx]]
    Klin = m.W[0] * B.T @ D @ B
    for model in MODELS:
        _, K, _, _ = _f(model, m, np.zeros_like(m.X), np.array([mu]), np.array([lam]))
        Kd = _dense(m, K)
        assert np.abs(Kd - Klin).max() < 1e-13 * np.abs(Klin).max()
        ev = np.linalg.eigvalsh(Kd)
        assert np.sum(np.abs(ev) < 1e-10 * ev.max()) == 6


@pytest.mark.parametrize("model", MODELS)
def test_uniaxial_energy_closed_form(model):
    """F = diag(s,1,1) on the unit cube: E = Psi(s) * volume, with
    StVK Psi = (mu + lam/2) e^2, e = (s^2-1)/2 and
    NH   Psi = mu/2 (s^2-1) - mu ln s + lam/2 (ln s)^2."""
    m = _mesh(lambda: M.kuhn6(3))
    mu, lam = 2.0, 3.0
    s = 1.13
    u = np.zeros_like(m.X)
    u[:, 0] = (s - 1.0) * m.X[:, 0]
    _, _, en, _ = _f(model, m, u, np.full(m.nt, mu), np.full(m.nt, lam))
    if model == "stvk":
        e = (s * s - 1) / 2
        psi = (mu + lam / 2) * e * e
    else:
        psi = mu / 2 * (s * s - 1) - mu * np.log(s) + lam / 2 * np.log(s) ** 2
    assert abs(en - psi) < 1e-13 * psi


@pytest.mark.parametrize("model", MODELS)
def test_patch_test_interior_forces_vanish(model):
    n = 4
    m = _mesh(lambda: M.kuhn6(n))
    A = np.array([[1.05, 0.02, -0.01], [0.03, 0.97, 0.04], [-0.02, 0.01, 1.08]])
    u = m.X @ A.T + np.array([0.1, -0.2, 0.3]) - m.X
    f, _, _, _ = _f(model, m, u, *_mat(m))
    ijk = np.rint(m.X * n).astype(int)
    interior = np.all((ijk > 0) & (ijk < n), axis=1)
    assert np.abs(f[interior]).max() < 1e-13 * np.abs(f).max()


def test_edge_matvec_equals_dense_fd_assembly():
    """5-tet cube: edge-relation matvec == dense K x, where dense K is built by
    central finite differences of the global force (no oracle K involved)."""
    m = _mesh(lambda: M.alt5(1))
    mu, lam = _mat(m)
    u = _rand_u(m.X, 4, 0.08)
    _, K, _, _ = _f("nh", m, u, mu, lam)
    eps = 1e-6
    J = np.zeros((3 * m.nv, 3 * m.nv))
    for v in range(m.nv):
        for a in range(3):
            up, um = u.copy(), u.copy()
            up[v, a] += eps
            um[v, a] -= eps
            J[:, 3 * v + a] = -(_f("nh", m, up, mu, lam)[0] - _f("nh", m, um, mu, lam)[0]).ravel() / (2 * eps)
    x = np.random.default_rng(5).uniform(-1, 1, size=(m.nv, 3))
    q = oracle.edge_matvec(m.row_ptr, m.head, K, x)
    ref = J @ x.ravel()
    assert np.abs(q.ravel() - ref).max() < 1e-7 * np.abs(ref).max()
    # and exactly the dense scatter of the same blocks (CSR traversal is total)
    assert np.abs(q.ravel() - _dense(m, K) @ x.ravel()).max() < 1e-14 * np.abs(ref).max()


def test_nh_inverted_element_flagged():
    m = _mesh(M.single_tet)
    u = np.zeros_like(m.X)
    u[3, 2] = -2.0                      # push apex through the base: J < 0
    f, K, en, inv = _f("nh", m, u, *_mat(m))
    assert inv == 1 and np.isnan(f).all()


def test_lame_conversion_inputs():
    mu, lam = S.lame(2e5, 0.3)
    assert abs(mu - 2e5 / 2.6) < 1e-9 and abs(lam - 2e5 * 0.3 / (1.3 * 0.4)) < 1e-9
