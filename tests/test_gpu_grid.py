"""GPU parity of the regular 2-D grid domain (P:733-772,
Fig. 3) against the oracle through the C ABI: affine-offset
stencils (incl. the 5-point Laplacian, shifts across the periodic wrap),
PointLocate (integer keys: bit-exact, decided in fp64 on both sides) and
Fig. 3's update_particle_vel.  Bars: fp64 1e-14 (stencil, interpolation),
fp32 1e-6."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1506_07577_b200 import ebb
    c = ebb.Context(0)
    yield c
    c.close()


def _rel(a, b):
    return np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-14), ("f32", 1e-6)])
@pytest.mark.parametrize("comps", [1, 2, 4])
def test_stencils(ctx, dtype, tol, comps):
    from paper_1506_07577_b200.grid import Grid2
    nx, ny = 173, 61                                    # ragged against the 32x8 blocks
    g = Grid2(ctx, nx, ny, name=f"gs{dtype}{comps}")
    f = np.random.default_rng(1).standard_normal((nx * ny, comps))
    if dtype == "f32":
        f = f.astype(np.float32).astype(np.float64)
    fin = g.cells.field("in", dtype, (comps, 1), init=f)
    fout = g.cells.field("out", dtype, (comps, 1))
    for off, w in ([[(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1)], [-4.0, 1.0, 1.0, 1.0, 1.0]],
                   [[(3, -2)], [1.0]],
                   [[(0, 0), (-5, 7), (nx + 1, -ny - 2), (2, 2)], [0.5, 0.25, -1.5, 2.0]]):
        g.stencil(fin, fout, off, w)
        ref = oracle.grid2_stencil(nx, ny, f, off, w)
        assert _rel(fout.read().reshape(nx * ny, comps), ref) <= tol


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-14), ("f32", 1e-6)])
def test_point_locate_and_particle_vel(ctx, dtype, tol):
    from paper_1506_07577_b200.grid import Grid2
    nx, ny, npart = 97, 45, 20_011
    g = Grid2(ctx, nx, ny, name=f"gp{dtype}")
    rng = np.random.default_rng(3)
    pos = np.zeros((npart, 3))
    pos[:, 0] = rng.uniform(-2.0, nx + 2.0, npart)        # outside the box too: periodic wrap
    pos[:, 1] = rng.uniform(-2.0, ny + 2.0, npart)
    pos[:, 2] = rng.uniform(-1, 1, npart)
    pos[:8, 0] = [0.5, 1.5, nx - 0.5, 0.5 + 1e-12, 0.5 - 1e-12, 10.0, 0.0, nx]   # cell centres, edges
    if dtype == "f32":
        pos = pos.astype(np.float32).astype(np.float64)
    P, pf, key = g.particles(f"parts{dtype}", pos, dtype=dtype)
    ref_key = oracle.grid2_point_locate(nx, ny, pos)
    assert np.array_equal(key.read().astype(np.int64).ravel(), ref_key)
    cv = rng.standard_normal((nx * ny, 2))
    if dtype == "f32":
        cv = cv.astype(np.float32).astype(np.float64)
    cvf = g.cells.field("vel", dtype, (2, 1), init=cv)
    vf = P.field("vel", dtype, (2, 1))
    g.particle_vel(key, cvf, pf, vf)
    ref = oracle.grid2_particle_vel(nx, ny, cv, pos, ref_key)
    assert _rel(vf.read().reshape(npart, 2), ref) <= tol


def test_grid_arguments_are_checked(ctx):
    from paper_1506_07577_b200.ebb import EbbError
    from paper_1506_07577_b200.grid import Grid2
    g = Grid2(ctx, 8, 8, name="gbad")
    a = g.cells.field("a", "f64")
    with pytest.raises(EbbError, match="EBB_E_PHASE"):
        g.stencil(a, a, [(1, 0)], [1.0])
    b = g.dual_cells.field("b", "f64")                  # wrong relation
    with pytest.raises(EbbError, match="EBB_E_TYPE"):
        g.stencil(a, b, [(1, 0)], [1.0])
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        g.stencil(a, g.cells.field("c", "f64"), [(0, 0)] * 17, [1.0] * 17)


def test_sorted_particles_keep_their_data(ctx):
    """ebb_sort_by_key_tuple on a 1-key field: particles reordered by dual
    cell (stable), every field permuted with them."""
    from paper_1506_07577_b200.grid import Grid2
    nx, ny, npart = 16, 12, 5000
    g = Grid2(ctx, nx, ny, name="gsort")
    rng = np.random.default_rng(9)
    pos = np.zeros((npart, 3))
    pos[:, 0] = rng.uniform(0, nx, npart)
    pos[:, 1] = rng.uniform(0, ny, npart)
    pos[:, 2] = np.arange(npart)                          # the original index rides along in z
    P, pf, key = g.particles("psort", pos)
    g.sort_particles(P, key)
    k = key.read().astype(np.int64).ravel()
    p2 = pf.read().reshape(npart, 3)
    ref = oracle.grid2_point_locate(nx, ny, pos)
    order = np.argsort(ref, kind="stable")
    assert np.array_equal(k, ref[order])
    assert np.array_equal(p2[:, 2].astype(np.int64), order)
