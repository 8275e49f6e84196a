"""Pins for the oracle's regular 2-D grid kernels (P:733-772 affine
indexing; Fig. 3): discrete Fourier modes are
eigenfunctions of the periodic 5-point Laplacian (closed-form eigenvalue),
hand-placed particles land in known dual cells (incl. the periodic wrap), and
bilinear interpolation reproduces affine velocity fields exactly."""
import numpy as np
import pytest

import oracle


def test_laplacian_of_a_fourier_mode_is_its_eigenvalue():
    nx, ny, kx, ky = 24, 16, 3, 2
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")     # (ny, nx): row-major i + nx j
    f = np.sin(2 * np.pi * kx * i / nx) * np.cos(2 * np.pi * ky * j / ny)
    off = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)]
    w = [-4.0, 1.0, 1.0, 1.0, 1.0]
    out = oracle.grid2_stencil(nx, ny, f.ravel()[:, None], off, w).ravel()
    lam = 2 * np.cos(2 * np.pi * kx / nx) - 2 + 2 * np.cos(2 * np.pi * ky / ny) - 2
    assert np.abs(out - lam * f.ravel()).max() <= 1e-13


def test_shift_stencil_is_a_periodic_translation():
    nx, ny = 7, 5
    f = np.random.default_rng(0).standard_normal((nx * ny, 2))
    out = oracle.grid2_stencil(nx, ny, f, [(2, -1)], [1.0])
    g = f.reshape(ny, nx, 2)
    assert np.array_equal(out.reshape(ny, nx, 2), np.roll(np.roll(g, -2, axis=1), 1, axis=0))


def test_point_locate_hand_cases():
    nx, ny = 8, 6
    pos = np.array([[2.75, 3.6, 0.0],      # a = floor(2.25) = 2, b = floor(3.1) = 3
                    [0.2, 0.4, 9.0],       # a = floor(-0.3) = -1 -> 7, b = -1 -> 5 (wrap)
                    [7.9, 5.5, 0.0],       # a = 7, b = 5
                    [1.5, 2.5, 0.0]])      # exactly on a cell centre: a = 1, b = 2
    d = oracle.grid2_point_locate(nx, ny, pos)
    assert list(d) == [2 + 8 * 3, 7 + 8 * 5, 7 + 8 * 5, 1 + 8 * 2]


@pytest.mark.parametrize("comps", [2, 3])
def test_bilinear_interpolation_is_exact_for_affine_fields(comps):
    """cell centres c_ij = (i + .5, j + .5); v(c) = A c + b; particles whose
    dual cell does not wrap get v(x, y) = A (x, y) + b."""
    nx, ny = 12, 9
    rng = np.random.default_rng(2)
    A = rng.standard_normal((comps, 2))
    b = rng.standard_normal(comps)
    i, j = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    cen = np.stack([i.ravel() + 0.5, j.ravel() + 0.5], 1)
    cell_vel = cen @ A.T + b
    pos = np.zeros((200, 3))
    pos[:, 0] = rng.uniform(0.5, nx - 0.5, 200)
    pos[:, 1] = rng.uniform(0.5, ny - 0.5, 200)
    d = oracle.grid2_point_locate(nx, ny, pos)
    vel = oracle.grid2_particle_vel(nx, ny, cell_vel, pos, d)
    assert np.abs(vel - (pos[:, :2] @ A.T + b)).max() <= 1e-12
    # a constant field is reproduced everywhere, including across the wrap
    pos[:, 0] = rng.uniform(0, nx, 200)
    pos[:, 1] = rng.uniform(0, ny, 200)
    d = oracle.grid2_point_locate(nx, ny, pos)
    const = oracle.grid2_particle_vel(nx, ny, np.tile(b, (nx * ny, 1)), pos, d)
    assert np.abs(const - b).max() <= 1e-14
