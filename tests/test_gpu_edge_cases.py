"""GPU parity on the degenerate and irregular inputs of the element map and
the solver (SURVEY §8(c) pins; tolerances of BASELINE.json north_star):

* the SPEC's 1-tet and 2-tet meshes for every scatter strategy;
* isolated vertices (referenced by no tet): zero force, zero stiffness row,
  the matvec's self-row-only vertex;
* a small C3-style blob (irregular boundary, vertices of low degree) for every
  strategy;
* no locality renumbering (vertices in scrambled order: tiny, ragged tiles);
* a vertex whose star exceeds the segmented map's per-tile instance cap is
  refused with EBB_E_RANGE, never silently mishandled;
* fp32 PCG iterates against the oracle fed the fp32-rounded system.
"""
import numpy as np
import pytest

import oracle
from helpers import rel_l2
from synth import mesh as M
from synth import state as S

pytestmark = pytest.mark.gpu

SCATTERS = {"atomic": 1, "segmented": 4, "color": 5, "chunk": 6, "chunk_red": 7}


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1506_07577_b200 import ebb
    c = ebb.Context(0)
    yield c
    c.close()


def _fem_and_oracle(ctx, X, tets, model, name, dtype="f64", renumber=True, seed=1):
    """GPU TetFEM and the oracle's map of the same input, both in stored order."""
    from paper_1506_07577_b200.tetfem import TetFEM
    rng = np.random.default_rng(seed)
    h = np.cbrt(np.abs(np.linalg.det(np.stack([X[tets[:, k]] - X[tets[:, 0]] for k in (1, 2, 3)], 1))).mean())
    u = 0.05 * X * np.array([1.0, -0.5, 0.3]) + rng.uniform(-0.03 * h, 0.03 * h, size=X.shape)
    mu, lam = S.materials(tets.shape[0], 2e5, 0.3, spread=0.1)
    if dtype == "f32":
        u = u.astype(np.float32).astype(np.float64)
        mu = mu.astype(np.float32).astype(np.float64)
        lam = lam.astype(np.float32).astype(np.float64)
    fem = TetFEM(ctx, X, tets, dtype=dtype, mu=mu, lam=lam, u=u, renumber=renumber, name=name)
    if renumber:
        new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
        order = np.argsort(new_of_old)
        Xn, un, mun, lamn = X[order], u[order], mu[tet_src], lam[tet_src]
    else:
        Xn, tets_new, un, mun, lamn = X, fem.v.read().astype(np.int64), u, mu, lam
    m = oracle.Mesh(Xn, tets_new)
    f, K, en, inv = oracle.element_map(model, m.X, un, m.tets, m.Dminv, m.W, mun, lamn, e=m.e, ne=m.ne)
    return fem, m, f, K, en


@pytest.mark.parametrize("scatter", list(SCATTERS))
@pytest.mark.parametrize("which", ["one", "two"])
def test_spec_tiny_meshes(ctx, which, scatter):
    X, tets = M.single_tet() if which == "one" else M.two_tets()
    fem, m, f, K, en = _fem_and_oracle(ctx, X, tets, "nh", f"tiny{which}{scatter}")
    assert fem.ne == (16 if which == "one" else 23)
    fem.map_forces("nh", scatter=SCATTERS[scatter])
    assert rel_l2(fem.f.read(), f) <= 1e-12
    assert rel_l2(fem.K.read(), K) <= 1e-12
    assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)


@pytest.mark.parametrize("scatter", list(SCATTERS))
def test_isolated_vertices(ctx, scatter):
    """Vertices no tet references: f = 0, their self row K = 0 (the relation
    keeps every vertex, P:797 caption: one self-loop edge per vertex)."""
    X, tets = M.kuhn6(3)
    extra = np.array([[2.0, 2.0, 2.0], [-1.0, 0.5, 0.5], [0.5, 3.0, 0.1]])
    X = np.vstack([X, extra])
    X, tets = M.permute_vertices(X, tets, 11)
    fem, m, f, K, en = _fem_and_oracle(ctx, X, tets, "stvk", f"iso{scatter}")
    fem.K.fill(7.0)                     # every row must be (over)written
    fem.f.fill(7.0)
    fem.map_forces("stvk", scatter=SCATTERS[scatter])
    Kg, fg = fem.K.read(), fem.f.read()
    assert rel_l2(fg, f) <= 1e-12 and rel_l2(Kg, K) <= 1e-12
    deg = np.bincount(m.tets.ravel(), minlength=m.X.shape[0])
    iso = np.nonzero(deg == 0)[0]
    assert iso.size == 3
    assert np.all(fg[iso] == 0.0)


@pytest.mark.parametrize("scatter", list(SCATTERS))
@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_small_blob(ctx, model, scatter):
    """Irregular C3-style mesh (metaball boundary, low-degree vertices)."""
    X, tets, n = M.blob(target_T=20_000)
    fem, m, f, K, en = _fem_and_oracle(ctx, X, tets, model, f"blob{model}{scatter}")
    fem.map_forces(model, scatter=SCATTERS[scatter])
    assert rel_l2(fem.f.read(), f) <= 1e-12
    assert rel_l2(fem.K.read(), K) <= 1e-12
    assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)


@pytest.mark.parametrize("scatter", ["segmented", "chunk", "chunk_red"])
def test_without_renumbering(ctx, scatter):
    """Scrambled vertex order (no SFC renumbering): tiles are ragged and
    tiny, the plan still covers every row exactly once."""
    X, tets = M.kuhn6(6)
    X, tets = M.permute_vertices(X, tets, 5)
    tets = M.permute_tets(tets, 6)
    fem, m, f, K, en = _fem_and_oracle(ctx, X, tets, "nh", f"noren{scatter}", renumber=False)
    fem.map_forces("nh", scatter=SCATTERS[scatter])
    assert rel_l2(fem.f.read(), f) <= 1e-12
    assert rel_l2(fem.K.read(), K) <= 1e-12


def _fan(k):
    """k tets around one hub vertex (a triangulated bipyramid fan)."""
    ang = 2 * np.pi * np.arange(k) / k
    ring = np.stack([np.cos(ang), np.sin(ang), np.zeros(k)], 1)
    X = np.vstack([[0.0, 0.0, 0.0], [0.0, 0.0, 1.0], ring])
    tets = np.array([[0, 2 + i, 2 + (i + 1) % k, 1] for i in range(k)], dtype=np.int64)
    d = np.einsum("ij,ij->i", X[tets[:, 1]] - X[tets[:, 0]],
                  np.cross(X[tets[:, 2]] - X[tets[:, 0]], X[tets[:, 3]] - X[tets[:, 0]]))
    tets[d < 0] = tets[d < 0][:, [0, 1, 3, 2]]
    return X, tets


def test_star_beyond_instance_cap(ctx, monkeypatch):
    """A vertex in 200 tets: fine with 256 instances per tile, EBB_E_RANGE with 128."""
    from paper_1506_07577_b200.ebb import EbbError
    X, tets = _fan(200)
    monkeypatch.setenv("EBB_SEG_NT", "256")
    fem, m, f, K, en = _fem_and_oracle(ctx, X, tets, "nh", "fan256")
    fem.map_forces("nh", scatter=SCATTERS["segmented"])
    assert rel_l2(fem.f.read(), f) <= 1e-12 and rel_l2(fem.K.read(), K) <= 1e-12
    monkeypatch.setenv("EBB_SEG_NT", "128")
    fem2, *_ = _fem_and_oracle(ctx, X, tets, "nh", "fan128")
    with pytest.raises(EbbError, match="EBB_E_RANGE"):
        fem2.map_forces("nh", scatter=SCATTERS["segmented"])


@pytest.mark.parametrize("variant", ["1", "2", "3"])
def test_pcg_fp32(ctx, variant, monkeypatch):
    """fp32 map + assembly + PCG (every variant) against the oracle's fp64
    step on the fp32-rounded inputs (the oracle never sees a GPU value):
    20 iterations agree to fp32 round-off amplified by the conditioning."""
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    from helpers import Case, gpu_fem, oracle_renumbered
    case = Case(n=5, model="nh")
    for a in ("u", "mu", "lam", "vel"):
        setattr(case, a, getattr(case, a).astype(np.float32).astype(np.float64))
    fem = gpu_fem(ctx, case, dtype="f32", name=f"pcg32{variant}")
    fem.map_forces("nh")
    fem.assemble(1e-2)
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], 1e-2, iters=20)
    fem.cg_init()
    fem.cg_step(20)
    assert rel_l2(fem.dv.read(), ref["dv"]) <= 1e-4


def test_plan_stats_and_cg_variant_queries(ctx):
    """ebb_map_plan_stats describes the plan the SEGMENTED map built (every tet
    is an instance of >= 1 tile; 10 block entries per tet); ebb_cg_variant
    resolves AUTO by the documented vertex-count rule."""
    from helpers import Case, gpu_fem
    case = Case(n=8, model="nh")
    fem = gpu_fem(ctx, case, name="stats")
    fem.map_forces("nh", scatter=SCATTERS["segmented"])
    st = fem.plan_stats()
    assert st["tiles"] >= 1 and st["instance_cap"] in (128, 256, 384, 512)
    assert st["instances"] >= fem.nt and st["redundancy"] >= 1.0
    assert st["entries"] >= 10 * fem.nt                       # + padding to 16 B per tile
    fem.assemble(1e-2)
    fem.cg_init()
    assert fem.cg_variant() == 2                               # 729 vertices <= 2.3e5
    from paper_1506_07577_b200 import _abi as A
    fem.cg.variant = A.CG_SAAD
    assert fem.cg_variant() == 1
    fem.cg.variant = A.CG_AUTO


def test_widening_entry_points_refuse_bad_arguments(ctx):
    """Argument checks of the §8(f) entry points: unknown rhs_form, a Newton
    assembly without v_n, a consistent mass on the wrong relation, a negative
    PCG tolerance, spring fields of mixed record shapes."""
    import ctypes as C

    from helpers import Case, gpu_fem
    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200.ebb import EbbError
    case = Case(n=3, model="nh")
    fem = gpu_fem(ctx, case, name="badargs")
    fem.map_forces("nh")
    d = A.ImplicitDesc()
    d.edges, d.K, d.A, d.self = fem.edges.h, fem.K.h, fem.K.h, fem.self_e.h
    d.mass, d.f, d.vel, d.b = fem.mass.h, fem.f.h, fem.vel.h, fem.b.h
    d.h = 1e-2
    d.rhs_form, d.vel0 = 7, A.NONE
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        ctx.check(ctx.L.ebb_implicit_assemble(ctx.h, C.byref(d), None))
    d.rhs_form = A.RHS_NEWTON
    with pytest.raises(EbbError):
        ctx.check(ctx.L.ebb_implicit_assemble(ctx.h, C.byref(d), None))
    wrong = fem.verts.field("me_wrong", "f64")                 # on verts, not on the edges
    with pytest.raises(EbbError, match="EBB_E_TYPE"):
        ctx.check(ctx.L.ebb_tetmesh_consistent_mass(ctx.h, fem.e.h, fem.W.h, 1e3, wrong.h, None))
    fem.assemble(1e-2)
    fem.cg_init()
    fem.cg.tol = -1.0
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        fem.cg_step(3)
    fem.cg.tol = 0.0
    from paper_1506_07577_b200.springmass import SpringMass
    sm = SpringMass(fem, name="badsp")
    f4 = fem.verts.field("f4", "f64", (4, 1))
    with pytest.raises(EbbError, match="EBB_E_TYPE"):
        ctx.check(ctx.L.ebb_spring_forces(ctx.h, fem.edges.h, sm.q.h, sm.rest_len.h, 1.0, f4.h, 0, None))


@pytest.mark.parametrize("nt", ["128", "256"])
def test_chunk_hub_vertex(ctx, nt, monkeypatch):
    """A vertex in 200 tets (and 300 with 128-tet tiles): its self row is summed
    from one to three tiles (messages from the earlier ones); the oracle's
    result either way.
    300 blocks of one row inside one 512-tet tile exceed the 8 x 31 chunk
    layout: EBB_E_RANGE, never a silent truncation."""
    from paper_1506_07577_b200.ebb import EbbError
    monkeypatch.setenv("EBB_CHUNK_NT", nt)
    for k in ((200, 300) if nt == "128" else (200,)):
        X, tets = _fan(k)
        fem, m, f, K, en = _fem_and_oracle(ctx, X, tets, "nh", f"fanchunk{nt}_{k}")
        for sc in ("chunk", "chunk_red"):          # messages / red.global.add into the hub's rows
            fem.map_forces("nh", scatter=SCATTERS[sc])
            assert rel_l2(fem.f.read(), f) <= 1e-12 and rel_l2(fem.K.read(), K) <= 1e-12
            assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)
    monkeypatch.setenv("EBB_CHUNK_NT", "512")
    X3, tets3 = _fan(300)
    fem3, *_ = _fem_and_oracle(ctx, X3, tets3, "nh", f"fanchunk300s_{nt}")
    with pytest.raises(EbbError, match="EBB_E_RANGE"):
        fem3.map_forces("nh", scatter=SCATTERS["chunk"])


def _pcg_case(ctx, X, tets, free, name, variant, iters, rho=1e3, noise=1e-3, ramp=None):
    """GPU map + assembly + PCG(iters) with the requested variant, and the
    oracle's implicit step (O9 + O10) on the same input, both in stored order."""
    from paper_1506_07577_b200.tetfem import TetFEM
    rng = np.random.default_rng(4)
    w = np.ones(X.shape[0]) if ramp is None else ramp     # smooth onset of the stretch off the fixed set
    u = (0.02 * X * np.array([1.0, -0.5, 0.3]) * w[:, None] + rng.uniform(-noise, noise, size=X.shape)) * free[:, None]
    mu, lam = S.materials(tets.shape[0], 2e5, 0.3, spread=0.1)
    fem = TetFEM(ctx, X, tets, dtype="f64", mu=mu, lam=lam, rho=rho, free=free, u=u, name=name)
    new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
    order = np.argsort(new_of_old)
    m = oracle.Mesh(X[order], tets_new, rho=rho)
    ref = oracle.implicit_step(m, "nh", u[order], np.zeros_like(u), mu[tet_src], lam[tet_src], free[order], 1e-2,
                               iters=iters)
    fem.map_forces("nh")
    fem.assemble(1e-2)
    fem.cg_init(variant=variant)
    fem.cg_step(iters)
    return fem, ref


@pytest.mark.parametrize("k", [200, 1500])
@pytest.mark.parametrize("variant", [1, 2, 3])
def test_pcg_hub_vertex(ctx, k, variant):
    """A hub vertex in k tets (a fan): the PCG stages are sized by the largest
    16-vertex chunk, not 16 x the longest group.  k = 200 fits every variant's
    TMA ring; k = 1500 (a 1,503-row group) fits none: single-reduction and
    symmetric resolve to Saad (reported by ebb_cg_variant), whose matvec then
    runs without staging (one warp per vertex).  Every case reproduces the
    oracle's 30 PCG iterations (<= 1e-8), never EBB_E_RANGE."""
    X, tets = _fan(k)
    ang = np.arctan2(X[:, 1], X[:, 0])
    free = (~((X[:, 2] == 0) & (np.abs(ang) < 0.6) & (np.hypot(X[:, 0], X[:, 1]) > 0.5))).astype(np.uint8)
    # sliver tets (ring spacing 2 pi / k): the stretch ramps in smoothly away
    # from the fixed arc and the noise stays far below the spacing
    ramp = np.clip((np.abs(ang) - 0.6) / 0.5, 0.0, 1.0)
    ramp[X[:, 2] != 0] = 1.0
    ramp[np.hypot(X[:, 0], X[:, 1]) < 0.5] = 1.0
    fem, ref = _pcg_case(ctx, X, tets, free, f"pcghub{k}_{variant}", variant, 30, noise=1e-5, ramp=ramp)
    assert np.isfinite(ref["dv"]).all() and ref["inverted"] == 0
    assert rel_l2(fem.dv.read(), ref["dv"]) <= 1e-8
    assert fem.cg_variant() == (variant if k == 200 else 1)


def test_matvec_hub_without_staging(ctx):
    """A 9,000-tet fan: the hub's group (9,003 rows) exceeds both the TMA
    stages and the register path's shared memory; ebb_map_edge_matvec runs
    the warp-per-vertex path and equals the oracle's edge-relation matvec."""
    X, tets = _fan(9000)
    fem, m, f, K, en = _fem_and_oracle(ctx, X, tets, "nh", "mvhub9000")
    rng = np.random.default_rng(8)
    fem.K.write(rng.uniform(-1, 1, size=(fem.ne, 9)))   # any matrix on the edge relation
    K = fem.K.read()
    p = rng.uniform(-1, 1, size=(fem.nv, 3))
    P = fem.verts.field("p_hub", "f64", (3, 1), init=p)
    Q = fem.verts.field("q_hub", "f64", (3, 1))
    fem.matvec(fem.K, P, Q)
    ref = oracle.edge_matvec(m.row_ptr, m.head, K, p)
    assert rel_l2(Q.read(), ref) <= 1e-13


@pytest.mark.parametrize("variant", [1, 2, 3])
def test_pcg_blob(ctx, variant):
    """C3-style blob (irregular metaball boundary, low-degree boundary
    vertices, ~20k tets): every PCG variant reproduces the oracle's 50
    iterations to <= 1e-8."""
    X, tets, n = M.blob(target_T=20_000)
    free = S.fixed_mask(X, n)
    fem, ref = _pcg_case(ctx, X, tets, free, f"pcgblob{variant}", variant, 50)
    assert rel_l2(fem.dv.read(), ref["dv"]) <= 1e-8


def _jacobi_condition(m, A, free):
    """kappa_2 of D^-1/2 A D^-1/2 on the free DOFs (dense; small meshes only)."""
    nv = m.nv
    Ad = np.zeros((3 * nv, 3 * nv))
    for v in range(nv):
        for e in range(m.row_ptr[v], m.row_ptr[v + 1]):
            Ad[3 * v:3 * v + 3, 3 * m.head[e]:3 * m.head[e] + 3] = A[e].reshape(3, 3)
    keep = np.repeat(np.asarray(free).astype(bool), 3)
    As = Ad[np.ix_(keep, keep)]
    d = 1.0 / np.sqrt(np.diag(As))
    ev = np.linalg.eigvalsh(d[:, None] * As * d[None, :])
    return ev[-1] / ev[0]


@pytest.mark.parametrize("variant", ["1", "2", "3"])
def test_pcg_fp32_50_iterations_derived_tolerance(ctx, variant, monkeypatch):
    """fp32 map + assembly + 50 PCG iterations (north_star's count) against the
    oracle's fp64 step on the fp32-rounded inputs.  The tolerance follows from
    the perturbation bound of a linear system, not a choice: the fp32 f and K
    carry at most the north_star fp32 bars (eps_b = eps_A = 1e-5 relative;
    b ~ h f here), so ||dv32 - dv64|| / ||dv64|| <= kappa (eps_A + eps_b) +
    40 kappa u (the recurrences' own rounding, u = 2^-24), with kappa the
    2-norm condition number of the Jacobi-scaled free-DOF system (entrywise
    relative perturbations), computed here."""
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    from helpers import Case, gpu_fem, oracle_renumbered
    case = Case(n=4, model="nh")
    for a in ("u", "mu", "lam", "vel"):
        setattr(case, a, getattr(case, a).astype(np.float32).astype(np.float64))
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], 1e-2, iters=50)
    kappa = _jacobi_condition(m, ref["A"], case.free[order])
    tol = kappa * (1e-5 + 1e-5) + 40.0 * kappa * 2.0 ** -24
    assert tol < 1e-3
    fem = gpu_fem(ctx, case, dtype="f32", name=f"pcg32d{variant}")
    fem.map_forces("nh")
    fem.assemble(1e-2)
    fem.cg_init()
    fem.cg_step(50)
    assert rel_l2(fem.dv.read(), ref["dv"]) <= tol


def test_field_read_async(ctx):
    """ebb_field_read_async: stream-ordered download into pinned memory
    (complete once the stream is synchronised); component-planar fields are
    refused (they need the synchronous layout conversion of ebb_field_read)."""
    import torch

    from paper_1506_07577_b200.ebb import EbbError
    R = ctx.relation("ra_async", 1000)
    x = np.random.default_rng(5).uniform(-1, 1, size=(1000, 3))
    f = R.field("x", "f64", (3, 1), init=x)
    out = torch.empty((1000, 3), dtype=torch.float64, pin_memory=True)
    s = torch.cuda.Stream()
    f.read_async(out.data_ptr(), x.nbytes, s)
    s.synchronize()
    assert np.array_equal(out.numpy(), x)
    g = R.field("y", "f64", (3, 1), "soa", init=x)
    with pytest.raises(EbbError, match="EBB_E_TYPE"):
        g.read_async(out.data_ptr(), x.nbytes, s)
