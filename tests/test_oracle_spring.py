"""Pins for the oracle's Fig. 2 spring-mass kernels.

Independent references: the 2-vertex chain integrated by hand (closed form of
one step), rest-state invariance, Newton's third law, the force as minus the
gradient of the spring potential by central finite differences, and energy
conservation of the Fig. 2 update over 1e4 steps.

Sign (DESIGN.md §3 reading 21): Fig. 2 prints v.force += K (rest_len dir - dq),
which is minus Hooke's force for K > 0; the oracle follows the print, so the
potential is U = -K/4 sum_directed (|dq| - L)^2 and a restoring spring has K < 0.
"""
import numpy as np
import pytest

import oracle
from synth import mesh as M


def _chain(delta):
    pos = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0]])
    q = np.array([[0.0, 0.0, 0.0], [1.0 + delta, 0.0, 0.0]])
    tail = np.array([0, 0, 1, 1])          # grouped by tail, self-loops kept (P:797 caption)
    head = np.array([0, 1, 0, 1])
    row_ptr = np.array([0, 2, 4])
    return pos, q, tail, head, row_ptr


def test_two_vertex_chain_one_step_by_hand():
    K, dt, delta, m = 1.0, 1e-4, 0.1, np.array([2.0, 3.0])
    pos, q, tail, head, row_ptr = _chain(delta)
    L = oracle.spring_init_len(tail, head, pos)
    assert np.array_equal(L, [0.0, 1.0, 1.0, 0.0])
    f = oracle.spring_forces(row_ptr, head, q, L, K)
    assert np.allclose(f, [[-K * delta, 0, 0], [K * delta, 0, 0]], rtol=0, atol=1e-15)
    qd = np.array([[0.0, 0.5, 0.0], [0.0, 0.0, -1.0]])
    q1, qd1, f1 = oracle.spring_apply(m, dt, q, qd, f)
    a = f / m[:, None]
    assert np.allclose(q1, q + qd * dt + 0.5 * a * dt * dt, rtol=0, atol=1e-16)
    assert np.allclose(qd1, qd + a * dt, rtol=0, atol=1e-16)
    assert np.all(f1 == 0.0)


def _mesh(n=3, seed=0):
    X, tets = M.kuhn6(n)
    m = oracle.Mesh(X, tets)
    rng = np.random.default_rng(seed)
    return m, rng


def test_rest_state_is_invariant():
    m, rng = _mesh()
    L = oracle.spring_init_len(m.tail, m.head, m.X)
    f = oracle.spring_forces(m.row_ptr, m.head, m.X, L, 1.0)
    assert np.abs(f).max() <= 1e-15
    q, qd = oracle.spring_steps(m.row_ptr, m.head, L, m.mass, 1.0, 1e-4, m.X, np.zeros_like(m.X), 100)
    assert np.abs(q - m.X).max() <= 1e-15 and np.abs(qd).max() <= 1e-12


def test_forces_sum_to_zero_and_are_minus_the_potential_gradient():
    m, rng = _mesh()
    L = oracle.spring_init_len(m.tail, m.head, m.X)
    q = m.X + rng.uniform(-0.05, 0.05, m.X.shape)
    K = 1.7
    f = oracle.spring_forces(m.row_ptr, m.head, q, L, K)
    assert np.abs(f.sum(0)).max() <= 1e-13 * np.abs(f).max()      # symmetric directed edges

    def U(qq):
        d = np.linalg.norm(qq[m.head] - qq[m.tail], axis=1)
        return -0.25 * K * np.sum((d - L) ** 2)

    eps = 1e-6
    for v, a in [(0, 0), (7, 1), (21, 2), (40, 0), (63, 2)]:
        qp, qm = q.copy(), q.copy()
        qp[v, a] += eps
        qm[v, a] -= eps
        fd = -(U(qp) - U(qm)) / (2 * eps)
        assert abs(fd - f[v, a]) <= 1e-7 * max(1.0, np.abs(f).max())


def test_energy_is_conserved_over_1e4_steps():
    """Restoring spring (K = -1 in the printed sign), 2-vertex chain, dt = 1e-4:
    kinetic + potential energy drifts < 1 % over 1e4 steps."""
    K, dt = -1.0, 1e-4
    pos, q, tail, head, row_ptr = _chain(0.1)
    m = np.array([1.0, 1.0])
    L = oracle.spring_init_len(tail, head, pos)
    qd = np.zeros_like(q)

    def energy(q, qd):
        d = np.linalg.norm(q[head] - q[tail], axis=1)
        return oracle.kinetic_energy(m, qd) - 0.25 * K * np.sum((d - L) ** 2)

    e0 = energy(q, qd)
    q, qd = oracle.spring_steps(row_ptr, head, L, m, K, dt, q, qd, 10_000)
    assert abs(energy(q, qd) - e0) <= 0.01 * e0
    assert oracle.kinetic_energy(m, qd) > 0.1 * e0      # it actually oscillated
