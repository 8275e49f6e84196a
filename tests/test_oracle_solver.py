"""Pins for oracle O8-O10 (explicit update, implicit assembly, Jacobi-PCG).

Independent references: a dense textbook PCG in numpy, numpy.linalg.solve,
the exact constant-acceleration solution (free fall) of both integrators,
and rest invariance.
"""
import numpy as np
import pytest

import oracle
from synth import mesh as M
from synth import state as S


def _dense(m, A):
    D = np.zeros((3 * m.nv, 3 * m.nv))
    for r in range(m.ne):
        a, b = m.tail[r], m.head[r]
        D[3 * a:3 * a + 3, 3 * b:3 * b + 3] = A[r]
    return D


def _system(n=2, model="nh", seed=7, h=1e-2, E=2e5, fixed=True):
    X, tets = M.kuhn6(n)
    m = oracle.Mesh(X, tets)
    free = S.fixed_mask(X, n) if fixed else np.ones(m.nv, np.uint8)
    u = S.stretch_noise_u(X, n, seed, free=free)
    v = np.random.default_rng(seed).uniform(-0.1, 0.1, size=X.shape) * free[:, None]
    mu, lam = S.materials(m.nt, E, 0.3)
    f, K, en, inv = oracle.element_map(model, m.X, u, m.tets, m.Dminv, m.W, mu, lam, e=m.e, ne=m.ne)
    A, b = oracle.implicit_assemble(m.row_ptr, m.head, K, m.mass, f, v, h, 0.1, 0.01)
    return m, free, u, v, f, K, A, b


def dense_pcg(A, b, mask, iters):
    """Textbook Jacobi-PCG (Saad Alg. 9.1) on a dense matrix with projection."""
    n = b.size
    d = np.diag(A).copy()
    x = np.zeros(n)
    r = b * mask
    z = np.where(mask > 0, r / d, 0.0)
    p = z.copy()
    rho = r @ z
    for _ in range(iters):
        q = (A @ p) * mask
        pq = p @ q
        al = rho / pq if pq != 0 else 0.0
        x += al * p
        r -= al * q
        z = np.where(mask > 0, r / d, 0.0)
        rn = r @ z
        be = rn / rho if rho != 0 else 0.0
        p = z + be * p
        rho = rn
    return x


def test_assembly_matches_dense_definition():
    m, free, u, v, f, K, A, b = _system()
    h, al, be = 1e-2, 0.1, 0.01
    Kd = _dense(m, K)
    Md = np.diag(np.repeat(m.mass, 3))
    Ad = Md + h * (al * Md + be * Kd) + h * h * Kd
    g = np.tile([0.0, -9.81, 0.0], m.nv)
    bd = h * (f.ravel() + Md @ g - (al * Md + be * Kd) @ v.ravel() - h * Kd @ v.ravel())
    assert np.abs(_dense(m, A) - Ad).max() < 1e-14 * np.abs(Ad).max()
    assert np.abs(b.ravel() - bd).max() < 1e-12 * np.abs(bd).max()


@pytest.mark.parametrize("iters", [1, 5, 20])
def test_pcg_matches_dense_textbook_pcg(iters):
    m, free, u, v, f, K, A, b = _system()
    mask = np.repeat(free, 3).astype(np.float64)
    x, hist, ns = oracle.pcg(m.row_ptr, m.head, A, b, free, iters)
    xd = dense_pcg(_dense(m, A), b.ravel(), mask, iters)
    assert np.abs(x.ravel() - xd).max() < 1e-11 * np.abs(xd).max()
    assert not ns


def test_pcg_converges_to_direct_solve():
    m, free, u, v, f, K, A, b = _system(n=2)
    idx = np.nonzero(np.repeat(free, 3))[0]
    Ad = _dense(m, A)[np.ix_(idx, idx)]
    assert np.linalg.eigvalsh(Ad).min() > 0               # SPD on free DOFs
    xs = np.linalg.solve(Ad, b.ravel()[idx])
    x, hist, ns = oracle.pcg(m.row_ptr, m.head, A, b, free, 3 * m.nv)
    assert np.abs(x.ravel()[idx] - xs).max() < 1e-10 * np.abs(xs).max()
    assert np.all(x[free == 0] == 0.0)


def test_explicit_rest_invariance():
    X, tets = M.kuhn6(3)
    m = oracle.Mesh(X, tets)
    mu, lam = S.materials(m.nt, 1e6, 0.3)
    u = np.zeros_like(X)
    v = np.zeros_like(X)
    for _ in range(5):
        u, v, f, en = oracle.explicit_step(m, "stvk", u, v, mu, lam, None, 1e-4, g=(0, 0, 0))
    assert np.all(u == 0) and np.all(v == 0)


def test_explicit_free_fall_exact():
    """Rigid translation under gravity: u_n = 1/2 g (n h)^2 (update P:376-377 is
    exact for constant acceleration; internal forces stay at round-off)."""
    X, tets = M.kuhn6(2)
    m = oracle.Mesh(X, tets)
    mu, lam = S.materials(m.nt, 1e6, 0.3)
    u = np.zeros_like(X)
    v = np.zeros_like(X)
    h, N = 1e-3, 10
    g = np.array([0.0, -9.81, 0.0])
    for _ in range(N):
        u, v, f, en = oracle.explicit_step(m, "stvk", u, v, mu, lam, None, h, g=g)
    assert np.abs(u - 0.5 * g * (N * h) ** 2).max() < 1e-12
    assert np.abs(v - g * N * h).max() < 1e-12


@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_implicit_free_fall(model):
    """Backward Euler from rest with no constraints: dv = h g exactly solves
    (M + h^2 K) dv = h M g because K annihilates translations."""
    X, tets = M.kuhn6(2)
    m = oracle.Mesh(X, tets)
    mu, lam = S.materials(m.nt, 2e5, 0.3)
    u = np.zeros_like(X)
    v = np.zeros_like(X)
    h = 1e-2
    out = oracle.implicit_step(m, model, u, v, mu, lam, None, h, iters=60)
    assert np.abs(out["dv"] - np.array([0, -9.81 * h, 0])).max() < 1e-8
    assert np.abs(out["u"] - h * out["v"]).max() < 1e-15


def test_pcg_zero_rhs_is_noop():
    m, free, u, v, f, K, A, b = _system()
    x, hist, ns = oracle.pcg(m.row_ptr, m.head, A, np.zeros_like(b), free, 10)
    assert np.all(x == 0) and np.all(hist == 0)


# ---------------------------------------------------------------- consistent mass
def _mass_dense(m, me):
    D = np.zeros((m.nv, m.nv))
    for r in range(m.ne):
        D[m.tail[r], m.head[r]] += me[r]
    return D


def test_consistent_mass_row_sums_are_the_lumped_mass():
    """sum_j rho W (1 + d_ij)/20 = rho W / 4: each row of the Galerkin mass sums
    to the lumped mass (orc_rest, an independent loop)."""
    X, tets = M.kuhn6(3)
    X = X + np.random.default_rng(3).uniform(-0.05, 0.05, X.shape) / 3 * (np.abs(X - 0.5) < 0.49)
    m = oracle.Mesh(X, tets, rho=7.5)
    me = oracle.consistent_mass(m.e, m.W, 7.5, m.ne)
    rows = np.add.reduceat(me, m.row_ptr[:-1])
    assert np.abs(rows - m.mass).max() <= 1e-14 * m.mass.max()
    assert np.all(me > 0)
    assert abs(me.sum() - 7.5 * 1.0) <= 1e-13               # rho * volume of the unit cube


@pytest.mark.parametrize("a,c", [((0.0, 0.0, 0.0), 1.0), ((1.0, -2.0, 0.5), 0.3), ((0.7, 0.0, -1.1), -2.0)])
def test_consistent_mass_integrates_quadratics_exactly(a, c):
    """phi^T M phi = rho * integral over [0,1]^3 of phi^2 for every affine phi
    (phi lies in the P1 space, M is its exact Gram matrix):
    int (a.x + c)^2 = sum a_i^2/3 + 2 sum_{i<j} a_i a_j/4 + c sum a_i + c^2.
    A wrong diagonal/off-diagonal split (e.g. rho W d_ij / 4) fails this."""
    X, tets = M.kuhn6(3)
    X = X + np.random.default_rng(4).uniform(-0.05, 0.05, X.shape) / 3 * (np.abs(X - 0.5) < 0.49)
    m = oracle.Mesh(X, tets, rho=2.0)
    me = oracle.consistent_mass(m.e, m.W, 2.0, m.ne)
    a = np.asarray(a)
    phi = m.X @ a + c
    quad = np.sum(a * a) / 3 + 0.5 * (a[0] * a[1] + a[0] * a[2] + a[1] * a[2]) + c * a.sum() + c * c
    got = np.sum(phi[m.tail] * me * phi[m.head])
    assert abs(got - 2.0 * quad) <= 1e-13 * max(1.0, abs(quad))
    # the lumped mass does NOT integrate a non-constant phi^2 exactly (the test discriminates)
    if np.any(a != 0):
        assert abs(np.sum(m.mass * phi * phi) - 2.0 * quad) > 1e-6


def test_consistent_assembly_matches_dense_definition():
    m, free, u, v, f, K, A, b = _system()
    me = oracle.consistent_mass(m.e, m.W, 1e3, m.ne)
    h, al, be = 1e-2, 0.1, 0.01
    A2, b2 = oracle.implicit_assemble_consistent(m.row_ptr, m.head, K, me, f, v, h, al, be)
    Kd = _dense(m, K)
    Md = np.kron(_mass_dense(m, me), np.eye(3))
    Ad = Md + h * (al * Md + be * Kd) + h * h * Kd
    g = np.tile([0.0, -9.81, 0.0], m.nv)
    bd = h * (f.ravel() + Md @ g - (al * Md + be * Kd) @ v.ravel() - h * Kd @ v.ravel())
    assert np.abs(_dense(m, A2) - Ad).max() < 1e-14 * np.abs(Ad).max()
    assert np.abs(b2.ravel() - bd).max() < 1e-12 * np.abs(bd).max()


@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_implicit_free_fall_consistent_mass(model):
    """(M + h^2 K) dv = h M g is solved by dv = h g for any SPD mass (K
    annihilates translations): the consistent-mass step falls freely too."""
    X, tets = M.kuhn6(2)
    m = oracle.Mesh(X, tets)
    mu, lam = S.materials(m.nt, 2e5, 0.3)
    u = np.zeros_like(X)
    v = np.zeros_like(X)
    out = oracle.implicit_step(m, model, u, v, mu, lam, None, 1e-2, iters=80, mass="consistent")
    assert np.abs(out["dv"] - np.array([0, -9.81e-2, 0])).max() < 1e-8


# ---------------------------------------------------------------- Newton iterations
def _newton_case(mass):
    X, tets = M.kuhn6(2)
    m = oracle.Mesh(X, tets)
    free = S.fixed_mask(X, 2)
    u = 2 * S.stretch_noise_u(X, 2, 5, free=free)          # large strain: visibly nonlinear
    v = np.random.default_rng(1).uniform(-0.5, 0.5, X.shape) * free[:, None]
    mu, lam = S.materials(m.nt, 2e5, 0.3)
    me = oracle.consistent_mass(m.e, m.W, m.rho, m.ne) if mass == "consistent" else oracle.lumped_as_edges(m)
    return m, free, u, v, mu, lam, me


def _be_residual(m, me, mu, lam, free, u0, v0, x, w, h, al, g=(0.0, -9.81, 0.0)):
    """Backward-Euler residual on the free DOFs, written from its definition
    with a dense mass: G = M (w - v_n)/h - f(x) - M g + alpha M w."""
    f, K, en, inv = oracle.element_map("nh", m.X, x, m.tets, m.Dminv, m.W, mu, lam, e=m.e, ne=m.ne)
    Md = _mass_dense(m, me)
    r = Md @ ((w - v0) / h) - f - Md @ np.tile(g, (m.nv, 1)) + al * (Md @ w)
    assert np.allclose(x, u0 + h * w, rtol=0, atol=1e-12)  # x = u_n + h w throughout
    return np.linalg.norm(r[free == 1])


@pytest.mark.parametrize("mass", ["lumped", "consistent"])
def test_newton_converges_quadratically(mass):
    """With converged linear solves (40 PCG iterations, r.z at 1e-12 of its
    start on these 81 DOFs), Newton's residual falls
    quadratically: G_{k+1} / G_k^2 stays constant.  A wrong right-hand side or
    Jacobian term would stall it (linear convergence or a wrong fixed point)."""
    m, free, u, v, mu, lam, me = _newton_case(mass)
    h, al = 0.05, 0.1
    G = []
    for k in range(1, 5):
        out = oracle.newton_step(m, "nh", u, v, mu, lam, free, h, iters=40, newton=k, alpha=al, mass=mass)
        assert not out["not_spd"]
        G.append(_be_residual(m, me, mu, lam, free, u, v, out["u"], out["v"], h, al))
    q = [G[k + 1] / G[k] ** 2 for k in range(3)]   # measured 4e-6..7e-6 (lumped)
    assert G[3] < 1e-8 * G[0]
    assert max(q) / min(q) < 10.0, (G, q)


def test_newton_one_iteration_is_the_linearised_step():
    m, free, u, v, mu, lam, me = _newton_case("lumped")
    a = oracle.newton_step(m, "stvk", u, v, mu, lam, free, 1e-2, iters=20, newton=1)
    b = oracle.implicit_step(m, "stvk", u, v, mu, lam, free, 1e-2, iters=20)
    assert np.array_equal(a["u"], b["u"]) and np.array_equal(a["v"], b["v"])


@pytest.mark.parametrize("mass", ["lumped", "consistent"])
def test_newton_free_fall(mass):
    """No constraints, at rest: every Newton iterate is the exact free fall
    (K annihilates translations): v = h g, u = h^2 g."""
    X, tets = M.kuhn6(2)
    m = oracle.Mesh(X, tets)
    mu, lam = S.materials(m.nt, 2e5, 0.3)
    z = np.zeros_like(X)
    out = oracle.newton_step(m, "nh", z, z, mu, lam, None, 1e-2, iters=80, newton=3, mass=mass)
    g = np.array([0.0, -9.81, 0.0])
    assert np.abs(out["v"] - 1e-2 * g).max() < 1e-8
    assert np.abs(out["u"] - 1e-4 * g).max() < 1e-10


@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_implicit_free_fall_multi_step(model):
    """The multi-step trajectory of the one-linearisation backward-Euler step
    (O9) against its closed form: from rest with no constraints every state
    is a rigid translation (f = 0, K annihilates it), so each step adds
    dv = h g exactly -- v_k = k h g, u_k = h^2 g k (k + 1) / 2 after k steps.
    A wrong state update (u += h v_old, a dropped v term of b) breaks it from
    step 2 on."""
    X, tets = M.kuhn6(2)
    m = oracle.Mesh(X, tets)
    mu, lam = S.materials(m.nt, 2e5, 0.3)
    u = np.zeros_like(X)
    v = np.zeros_like(X)
    h, N = 1e-2, 10
    g = np.array([0.0, -9.81, 0.0])
    for _ in range(N):
        out = oracle.implicit_step(m, model, u, v, mu, lam, None, h, iters=120)
        u, v = out["u"], out["v"]
    assert np.abs(v - N * h * g).max() < 1e-8
    assert np.abs(u - h * h * g * N * (N + 1) / 2).max() < 1e-9


def _total_energy(m, model, u, v, mu, lam):
    f, K, en, inv = oracle.element_map(model, m.X, u, m.tets, m.Dminv, m.W, mu, lam, e=m.e, ne=m.ne, want_K=False)
    return 0.5 * float(np.sum(m.mass[:, None] * v * v)) + float(en)


@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_backward_euler_dissipates_energy(model):
    """A multi-step property of converged backward Euler on a conservative
    system (no gravity, no damping, fixed walls): with M (v' - v) = h f(u'),
    u' - u = h v' and f = -grad Psi, the total energy changes by
    Psi(u') - Psi(u) - grad Psi(u').(u' - u) - |v' - v|_M^2 / 2, which is
    <= 0 wherever Psi is convex along the step -- true near the rest state
    (small strain).  Converged Newton (4 iterations, 300 PCG iterations)
    makes the oracle's trajectory the backward-Euler one; a wrong sign of a
    force or stiffness term, or a wrong mass, makes the energy grow."""
    X, tets = M.kuhn6(3)
    m = oracle.Mesh(X, tets)
    free = S.fixed_mask(X, 3)
    u = 1e-3 * np.random.default_rng(4).uniform(-1, 1, X.shape) * free[:, None]
    v = np.zeros_like(X)
    mu, lam = S.materials(m.nt, 2e5, 0.3)
    E = [_total_energy(m, model, u, v, mu, lam)]
    for _ in range(12):
        out = oracle.newton_step(m, model, u, v, mu, lam, free, 2e-3, iters=300, newton=4, g=(0.0, 0.0, 0.0))
        u, v = out["u"], out["v"]
        E.append(_total_energy(m, model, u, v, mu, lam))
    dE = np.diff(E)
    assert np.all(dE <= 1e-12 * E[0]), dE / E[0]
    assert E[-1] < 0.999 * E[0]                  # and it does dissipate
