"""GPU parity of the element map (a4-a8) against the oracle (O6/O7).

Bars (BASELINE.json north_star): fp64 forces relative L2 <= 1e-12; fp32 <= 1e-5
with the oracle fed the fp32-rounded inputs.  The same bars are applied to the
stiffness (relative L2 over all blocks) and the strain energy.
"""
import numpy as np
import pytest

import oracle
from helpers import Case, gpu_fem, oracle_renumbered, rel_l2

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


def _oracle_map(case, m, order, tet_src, model, u=None):
    u = case.u[order] if u is None else u
    return oracle.element_map(model, m.X, u, m.tets, m.Dminv, m.W, case.mu[tet_src], case.lam[tet_src],
                              e=m.e, ne=m.ne)


SCATTERS = {"atomic": 1, "segmented": 4, "color": 5, "chunk": 6, "chunk_red": 7}


@pytest.mark.parametrize("scatter", ["atomic", "segmented", "color", "chunk", "chunk_red"])
@pytest.mark.parametrize("model", ["stvk", "nh"])
@pytest.mark.parametrize("n,mesh", [(4, "kuhn6"), (9, "kuhn6"), (4, "alt5")])
def test_map_fp64(ctx, model, n, mesh, scatter):
    case = Case(n=n, mesh=mesh, model=model, spread=0.1)
    fem = gpu_fem(ctx, case, name=f"m64{model}{n}{mesh}{scatter}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, model)
    fem.map_forces(model, scatter=SCATTERS[scatter])
    assert rel_l2(fem.f.read(), f) <= 1e-12
    assert rel_l2(fem.K.read(), K) <= 1e-12
    assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)
    assert ctx.error_counts(reset=True)["inverted"] == 0


@pytest.mark.parametrize("scatter", ["atomic", "segmented", "color", "chunk", "chunk_red"])
@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_map_fp32_displacement_form(ctx, model, scatter):
    case = Case(n=8, model=model, spread=0.1)
    # oracle is fed the fp32-rounded inputs
    case.u = case.u.astype(np.float32).astype(np.float64)
    case.mu = case.mu.astype(np.float32).astype(np.float64)
    case.lam = case.lam.astype(np.float32).astype(np.float64)
    fem = gpu_fem(ctx, case, dtype="f32", name=f"m32{model}{scatter}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, model)
    fem.map_forces(model, scatter=SCATTERS[scatter])
    assert rel_l2(fem.f.read(), f) <= 1e-5
    assert rel_l2(fem.K.read(), K) <= 1e-5
    assert abs(fem.energy.get() - en) <= 1e-5 * abs(en)


def test_map_small_strain_fp32(ctx):
    """1e-3 strain: the displacement form keeps fp32 within 1e-5."""
    case = Case(n=6, model="nh")
    case.u = (case.u * 0.01).astype(np.float32).astype(np.float64)
    fem = gpu_fem(ctx, case, dtype="f32", name="m32small")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, "nh")
    fem.map_forces("nh")
    assert rel_l2(fem.f.read(), f) <= 1e-5


def test_map_rest_state_is_zero(ctx):
    case = Case(n=3)
    case.u[:] = 0.0
    fem = gpu_fem(ctx, case, name="mrest")
    fem.map_forces("nh")
    assert np.abs(fem.f.read()).max() == 0.0 and fem.energy.get() == 0.0


def test_map_inverted_element_counted(ctx):
    case = Case(n=2, order_seed=None)
    fem = gpu_fem(ctx, case, renumber=False, name="minv")
    u = case.u.copy()
    u[:] = 0.0
    u[:, 0] = -2.0 * case.X[:, 0]            # mirror x: every tet inverted
    fem.u.write(u)
    ctx.error_counts(reset=True)
    fem.map_forces("nh")
    assert ctx.error_counts(reset=True)["inverted"] == fem.nt


def test_map_energy_deterministic(ctx):
    case = Case(n=6)
    fem = gpu_fem(ctx, case, name="mdet")
    fem.map_forces("nh")
    e1 = fem.energy.get()
    fem.map_forces("nh")
    assert fem.energy.get() == e1


@pytest.mark.parametrize("scatter", ["atomic", "segmented", "color", "chunk", "chunk_red"])
def test_map_accumulates_without_zeroing(ctx, scatter):
    """zero_outputs = 0 is the paper's `+=` into existing fields."""
    case = Case(n=4, model="stvk")
    fem = gpu_fem(ctx, case, name=f"macc{scatter}")
    fem.map_forces("stvk", scatter=SCATTERS[scatter])
    f1, K1 = fem.f.read(), fem.K.read()
    fem.map_forces("stvk", scatter=SCATTERS[scatter], zero_outputs=False)
    assert rel_l2(fem.f.read(), 2 * f1) <= 1e-14
    assert rel_l2(fem.K.read(), 2 * K1) <= 1e-14


def test_segmented_map_is_bitwise_deterministic(ctx):
    """The segmented strategy has no atomics: reruns are bitwise identical."""
    case = Case(n=8, model="nh")
    fem = gpu_fem(ctx, case, name="mdet4")
    fem.map_forces("nh", scatter=SCATTERS["segmented"])
    f1, K1 = fem.f.read(), fem.K.read()
    fem.map_forces("nh", scatter=SCATTERS["segmented"])
    assert np.array_equal(fem.f.read(), f1) and np.array_equal(fem.K.read(), K1)


@pytest.mark.parametrize("nt", ["256", "384", "512"])
@pytest.mark.parametrize("model,dtype", [("nh", "f64"), ("stvk", "f64"), ("nh", "f32")])
def test_segmented_tile_caps(ctx, nt, model, dtype, monkeypatch):
    """Every instance cap (threads per CTA) gives the oracle's result: many
    small ragged tiles (n=9 -> 6000 tets over ~25-60 tiles)."""
    monkeypatch.setenv("EBB_SEG_NT", nt)
    case = Case(n=9, model=model, spread=0.1)
    if dtype == "f32":
        case.u = case.u.astype(np.float32).astype(np.float64)
        case.mu = case.mu.astype(np.float32).astype(np.float64)
        case.lam = case.lam.astype(np.float32).astype(np.float64)
    fem = gpu_fem(ctx, case, dtype=dtype, name=f"mseg{nt}{model}{dtype}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, model)
    fem.map_forces(model, scatter=SCATTERS["segmented"])
    tol = 1e-12 if dtype == "f64" else 1e-5
    assert rel_l2(fem.f.read(), f) <= tol
    assert rel_l2(fem.K.read(), K) <= tol
    assert abs(fem.energy.get() - en) <= tol * abs(en)


@pytest.mark.parametrize("grid", ["1", "3"])
def test_segmented_long_tile_runs(ctx, grid, monkeypatch):
    """A few CTAs walking hundreds of consecutive tiles each (descriptor ring
    refilled every 32 tiles, entry buffers and the register pipeline wrapping
    many times) give the oracle's result."""
    monkeypatch.setenv("EBB_SEG_GRID", grid)
    case = Case(n=16, model="nh", spread=0.1)
    fem = gpu_fem(ctx, case, name=f"mseggrid{grid}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, "nh")
    fem.map_forces("nh", scatter=SCATTERS["segmented"])
    assert rel_l2(fem.f.read(), f) <= 1e-12
    assert rel_l2(fem.K.read(), K) <= 1e-12
    assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)


def test_color_map_is_bitwise_deterministic(ctx):
    """The coloured strategy has no atomics: reruns are bitwise identical."""
    case = Case(n=8, model="nh")
    fem = gpu_fem(ctx, case, name="mdet5")
    fem.map_forces("nh", scatter=SCATTERS["color"])
    f1, K1 = fem.f.read(), fem.K.read()
    fem.map_forces("nh", scatter=SCATTERS["color"])
    assert np.array_equal(fem.f.read(), f1) and np.array_equal(fem.K.read(), K1)


def test_chunk_map_is_bitwise_deterministic(ctx):
    """The chunk strategy sums in plan order (own blocks, then the messages by
    sender tile) whatever the timing: reruns are bitwise identical."""
    case = Case(n=12, model="nh")
    fem = gpu_fem(ctx, case, name="mdet6")
    fem.map_forces("nh", scatter=SCATTERS["chunk"])
    f1, K1, e1 = fem.f.read(), fem.K.read(), fem.energy.get()
    for _ in range(3):
        fem.map_forces("nh", scatter=SCATTERS["chunk"])
        assert np.array_equal(fem.f.read(), f1) and np.array_equal(fem.K.read(), K1)
        assert fem.energy.get() == e1


@pytest.mark.parametrize("scatter", ["chunk", "chunk_red"])
@pytest.mark.parametrize("nt", ["128", "256", "384", "512"])
@pytest.mark.parametrize("model,dtype", [("nh", "f64"), ("stvk", "f64"), ("nh", "f32"), ("stvk", "f32")])
def test_chunk_tile_sizes(ctx, nt, model, dtype, monkeypatch, scatter):
    """Every tile size (tets per CTA) gives the oracle's result: n=9 -> 4374
    tets over 9..35 tiles, the last one ragged, rows spanning many tiles."""
    monkeypatch.setenv("EBB_CHUNK_NT", nt)
    case = Case(n=9, model=model, spread=0.1)
    if dtype == "f32":
        case.u = case.u.astype(np.float32).astype(np.float64)
        case.mu = case.mu.astype(np.float32).astype(np.float64)
        case.lam = case.lam.astype(np.float32).astype(np.float64)
    fem = gpu_fem(ctx, case, dtype=dtype, name=f"mchunk{nt}{model}{dtype}{scatter}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, model)
    fem.map_forces(model, scatter=SCATTERS[scatter])
    tol = 1e-12 if dtype == "f64" else 1e-5
    assert rel_l2(fem.f.read(), f) <= tol
    assert rel_l2(fem.K.read(), K) <= tol
    assert abs(fem.energy.get() - en) <= tol * abs(en)


@pytest.mark.parametrize("grid", ["1", "2", "5"])
def test_chunk_few_ctas(ctx, grid, monkeypatch):
    """One CTA (every tile processed in order by itself: its messages are all
    from its own earlier tiles) and a few CTAs claiming hundreds of tiles each
    (tile queue, entry buffers and the register pipeline wrapping many times)
    give the oracle's result, bitwise equal to the full grid."""
    case = Case(n=16, model="nh", spread=0.1)
    fem = gpu_fem(ctx, case, name=f"mchunkgrid{grid}")
    fem.map_forces("nh", scatter=SCATTERS["chunk"])
    f_full, K_full = fem.f.read(), fem.K.read()
    monkeypatch.setenv("EBB_CHUNK_GRID", grid)
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, "nh")
    fem.map_forces("nh", scatter=SCATTERS["chunk"])
    assert rel_l2(fem.f.read(), f) <= 1e-12
    assert rel_l2(fem.K.read(), K) <= 1e-12
    assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)
    assert np.array_equal(fem.f.read(), f_full) and np.array_equal(fem.K.read(), K_full)


def test_chunk_plan_stats(ctx):
    """The CHUNK plan computes every tet once: 10 block entries per tet over
    ceil(T / NT) tiles; messages are the segments of rows owned by a later
    tile (fewer than the segments); the plan is built on the device."""
    case = Case(n=10, model="nh")
    fem = gpu_fem(ctx, case, name="chunkstats")
    fem.map_forces("nh", scatter=SCATTERS["chunk"])
    st = fem.chunk_stats()
    assert st["tets_per_tile"] in (128, 256, 384, 512)
    assert st["tiles"] == -(-fem.nt // int(st["tets_per_tile"]))
    assert (fem.ne + fem.nv) // 2 <= st["segments"] <= 10 * fem.nt   # >= one per canonical row
    assert 0 < st["messages"] < st["segments"]
    assert st["zero_rows"] == 0 and st["plan_bytes_per_tet"] > 0


@pytest.mark.parametrize("model,dtype", [("nh", "f64"), ("stvk", "f64"), ("nh", "f32")])
@pytest.mark.parametrize("mesh", ["kuhn", "blob", "noren"])
def test_segmented_plan_device_equals_host(ctx, model, dtype, mesh, monkeypatch):
    """The SEGMENTED plan built on the device (seg_plan.cu) is the host
    builder's plan word for word: same statistics, and the map run with either
    plan gives bitwise-identical f, K and energy (the kernel is deterministic
    in its plan).  Meshes: renumbered Kuhn cube, the irregular blob, and a
    scrambled (unrenumbered) cube with ragged tiles."""
    from synth import mesh as M
    from paper_1506_07577_b200.tetfem import TetFEM
    if mesh == "kuhn":
        X, tets = M.kuhn6(12)
    elif mesh == "blob":
        X, tets, _ = M.blob(target_T=30_000)
    else:
        X, tets = M.kuhn6(8)
        X, tets = M.permute_vertices(X, tets, 5)
        tets = M.permute_tets(tets, 6)
    rng = np.random.default_rng(3)
    u = 0.02 * X * np.array([1.0, -0.5, 0.3]) + rng.uniform(-1e-3, 1e-3, size=X.shape)
    from synth import state as S
    mu, lam = S.materials(tets.shape[0], 2e5, 0.3, spread=0.1)
    out = []
    for which in ("device", "host"):
        monkeypatch.setenv("EBB_SEG_PLAN", which)
        fem = TetFEM(ctx, X, tets, dtype=dtype, mu=mu, lam=lam, u=u, renumber=(mesh != "noren"),
                     name=f"pl{model}{dtype}{mesh}{which}")
        fem.map_forces(model, scatter=SCATTERS["segmented"])
        st = fem.plan_stats()
        out.append((st, fem.f.read(), fem.K.read(), fem.energy.get()))
    (sd, fd, Kd, ed), (sh, fh, Kh, eh) = out
    for k in ("tiles", "instances", "entries", "items", "instance_cap", "max_tile_entries"):
        assert sd[k] == sh[k], k
    assert np.array_equal(fd, fh) and np.array_equal(Kd, Kh) and ed == eh


@pytest.mark.parametrize("sid", [2, 3])
def test_retired_strategies_refused(ctx, sid):
    """TILED (2) and GATHER (3) were retired in round 2 (measured slower than
    SEGMENTED at every size): EBB_E_ARG, never a silent substitute."""
    from paper_1506_07577_b200.ebb import EbbError
    fem = gpu_fem(ctx, Case(n=3), name=f"retired{sid}")
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        fem.map_forces("nh", scatter=sid)


@pytest.mark.parametrize("grid", ["1", "3"])
def test_chunk_red_few_ctas_and_repeat(ctx, grid, monkeypatch):
    """The RED mode of the chunk map (SURVEY strategy (i): rows fed by several
    tiles zeroed, then red.global.add) on one and three CTAs and on the full
    grid, twice in a row (the shared rows are re-zeroed every launch): the
    oracle's result each time (no bitwise claim: RED order varies)."""
    case = Case(n=12, model="nh", spread=0.1)
    fem = gpu_fem(ctx, case, name=f"mchunkred{grid}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = _oracle_map(case, m, order, tet_src, "nh")
    for env in (None, grid):
        if env:
            monkeypatch.setenv("EBB_CHUNK_GRID", env)
        for _ in range(2):
            fem.map_forces("nh", scatter=SCATTERS["chunk_red"])
            assert rel_l2(fem.f.read(), f) <= 1e-12
            assert rel_l2(fem.K.read(), K) <= 1e-12
            assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)
