"""GPU parity of the edge matvec (a10), global reductions (a8), implicit assembly
(a9), Jacobi-PCG (a11-a12) and both integrators against the oracle.

Bars: CG iterates <= 1e-8 relative after 50 iterations (fp64, north_star);
explicit steps <= 1e-12 (fp64) per step; matvec <= 1e-13 (fp64), 1e-6 (fp32).
"""
import json
import os

import numpy as np
import pytest

import oracle
from helpers import Case, gpu_fem, oracle_renumbered, rel_l2

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1506_07577_b200 import ebb
    c = ebb.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-13), ("f32", 1e-6)])
def test_edge_matvec(ctx, dtype, tol):
    case = Case(n=7)
    fem = gpu_fem(ctx, case, dtype=dtype, name=f"mv{dtype}")
    m, *_ = oracle_renumbered(case)
    rng = np.random.default_rng(6)
    A = rng.uniform(-1, 1, size=(m.ne, 3, 3))
    p = rng.uniform(-1, 1, size=(m.nv, 3))
    if dtype == "f32":
        A = A.astype(np.float32).astype(np.float64)
        p = p.astype(np.float32).astype(np.float64)
    fem.K.write(A)
    P = fem.verts.field("p_mv", dtype, (3, 1), init=p)
    Q = fem.verts.field("q_mv", dtype, (3, 1))
    fem.matvec(fem.K, P, Q)
    ref = oracle.edge_matvec(m.row_ptr, m.head, A, p)
    assert rel_l2(Q.read(), ref) <= tol
    # masked + fused p.q (global `+=`)
    pq = ctx.global_(f"pq_{dtype}")
    fem.matvec(fem.K, P, Q, mask=True, pq=pq)
    free = fem.free.read()
    refm = ref * free[:, None]
    assert rel_l2(Q.read(), refm) <= tol
    assert abs(pq.get() - oracle.dot(p, refm)) <= 10 * tol * np.abs(p).sum() * np.abs(refm).max()


def test_global_reduce_ops(ctx):
    from paper_1506_07577_b200 import _abi as A
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    R = ctx.relation("red", 4)
    x = R.field("x", "f64", init=g["global_sum"]["values"])
    out = ctx.global_("red_out")
    for op, want in ((A.RED_SUM, 10.0), (A.RED_MAX, 6.0), (A.RED_MIN, 0.0)):
        ctx.check(ctx.L.ebb_global_reduce(ctx.h, op, x.h, A.NONE, A.NONE, out.h, None))
        assert out.get() == want
    # S:295 measureTotalEnergy: E = sum 1/2 m qd.qd = 3.0, as a DOT of (m/2 qd) and qd
    e = g["global_energy"]
    V = ctx.relation("red.v", 3)
    qd = np.array(e["qd"], dtype=np.float64)
    a = V.field("a", "f64", (3, 1), init=0.5 * np.array(e["mass"])[:, None] * qd)
    b = V.field("b", "f64", (3, 1), init=qd)
    ctx.check(ctx.L.ebb_global_reduce(ctx.h, A.RED_DOT, a.h, b.h, A.NONE, out.h, None))
    assert out.get() == e["E"]


def test_global_reduce_large_masked(ctx):
    from paper_1506_07577_b200 import _abi as A
    n = 1_000_003
    rng = np.random.default_rng(1)
    x = rng.standard_normal((n, 3))
    mk = (rng.random(n) < 0.7).astype(np.uint8)
    R = ctx.relation("redL", n)
    fx = R.field("x", "f64", (3, 1), init=x)
    fm = R.field("m", "u8", init=mk)
    out = ctx.global_("redL_out")
    ctx.check(ctx.L.ebb_global_reduce(ctx.h, A.RED_DOT, fx.h, fx.h, fm.h, out.h, None))
    ref = float(np.sum(x[mk == 1] ** 2))
    assert abs(out.get() - ref) <= 1e-12 * ref
    v1 = out.get()
    ctx.check(ctx.L.ebb_global_reduce(ctx.h, A.RED_DOT, fx.h, fx.h, fm.h, out.h, None))
    assert out.get() == v1                          # deterministic two-pass
    ctx.check(ctx.L.ebb_global_reduce(ctx.h, A.RED_MAX, fx.h, A.NONE, A.NONE, out.h, None))
    assert out.get() == x.max()


@pytest.mark.parametrize("variant", ["1", "2", "3"])
@pytest.mark.parametrize("model", ["nh", "stvk"])
def test_implicit_step(ctx, model, variant, monkeypatch):
    """Every PCG variant (1 = Saad Alg. 9.1, 2 = single-reduction
    Chronopoulos-Gear, 3 = Saad on the symmetric half of A with red.add
    transposes) reproduces the oracle's Saad iterates after 50 its."""
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    case = Case(n=6, model=model, vel_amp=0.05)
    h, iters, al, be = 1e-2, 50, 0.05, 0.002
    fem = gpu_fem(ctx, case, name=f"imp{model}{variant}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    out = oracle.implicit_step(m, model, case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], h, iters=iters, alpha=al, beta=be)
    fem.implicit_step(model, h=h, iters=iters, alpha=al, beta=be)
    assert rel_l2(fem.b.read(), out["b"]) <= 1e-12
    assert rel_l2(fem.K.read(), out["A"]) <= 1e-12          # A assembled in place of K
    assert rel_l2(fem.dv.read(), out["dv"]) <= 1e-8
    assert rel_l2(fem.vel.read(), out["v"]) <= 1e-8
    assert rel_l2(fem.u.read(), out["u"]) <= 1e-8
    assert abs(fem.cg_rho() - out["rho"][-1]) <= 1e-6 * abs(out["rho"][0])
    assert ctx.error_counts(reset=True)["not_spd"] == 0


def test_explicit_C1(ctx):
    """BASELINE configs[0]: StVK explicit, 4x4x4 Kuhn cube (384 tets), fp64, 10 steps."""
    case = Case(n=4, model="stvk", E=1e6)
    h = 1e-4
    fem = gpu_fem(ctx, case, name="C1")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    u, v = case.u[order], case.vel[order]
    mu, lam, free = case.mu[tet_src], case.lam[tet_src], case.free[order]
    for step in range(10):
        u, v, f, en = oracle.explicit_step(m, "stvk", u, v, mu, lam, free, h)
        fem.explicit_step("stvk", h=h)
        assert rel_l2(fem.u.read(), u) <= 1e-12, step
        assert rel_l2(fem.vel.read(), v) <= 1e-12, step
        assert abs(fem.energy.get() - en) <= 1e-12 * abs(en)


@pytest.mark.parametrize("variant", ["1", "2", "3"])
def test_cg_zero_rhs_noop(ctx, variant, monkeypatch):
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    case = Case(n=3)
    fem = gpu_fem(ctx, case, name=f"cg0{variant}")
    fem.map_forces("nh")
    fem.assemble(1e-2)
    fem.b.fill(0.0)
    fem.cg_init()
    fem.cg_step(5)
    assert np.all(fem.dv.read() == 0.0) and fem.cg_rho() == 0.0


@pytest.mark.parametrize("variant", ["1", "2", "3"])
def test_C2_full_size_implicit_step(ctx, variant, monkeypatch):
    """BASELINE configs[1] at full size (998,250 tets), bench launch configuration:
    integer maps bit-exact, f/K <= 1e-12, CG iterate <= 1e-8 after 50 iterations."""
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    case = Case(n=55, model="nh", E=2e5)
    fem = gpu_fem(ctx, case, name=f"C2v{variant}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    assert np.array_equal(fem.vert_order(), order)
    assert np.array_equal(fem.tet_order(), tet_src)
    assert np.array_equal(fem.head.read(), m.head)
    out = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], 1e-2, iters=50)
    fem.implicit_step("nh", h=1e-2, iters=50)
    assert rel_l2(fem.f.read(), out["f"]) <= 1e-12
    assert rel_l2(fem.K.read(), out["A"]) <= 1e-12
    assert rel_l2(fem.dv.read(), out["dv"]) <= 1e-8
    assert ctx.error_counts(reset=True) == dict(inverted=0, not_spd=0, bounds=0, peer_timeouts=0)


def test_graph_capture_replays_the_step(ctx):
    """ebb_graph_* capture of one implicit step replays to the eager result."""
    import torch
    case = Case(n=5, model="nh", vel_amp=0.02)
    s = torch.cuda.Stream()
    a = gpu_fem(ctx, case, name="geager")
    b = gpu_fem(ctx, case, name="ggraph")
    for fem in (a, b):                      # warm-up: plans and work fields
        fem.implicit_step("nh", h=1e-2, iters=20, stream=s)
    s.synchronize()
    ctx.graph_begin(s)
    b.implicit_step("nh", h=1e-2, iters=20, stream=s)
    g = ctx.graph_end(s)
    for _ in range(3):
        a.implicit_step("nh", h=1e-2, iters=20, stream=s)
        ctx.graph_launch(g, s)
    s.synchronize()
    assert rel_l2(b.u.read(), a.u.read()) <= 1e-12
    assert rel_l2(b.dv.read(), a.dv.read()) <= 1e-12


@pytest.mark.parametrize("variant", ["1", "2", "3"])
@pytest.mark.parametrize("iters", [1, 5, 20])
def test_cg_iterates_and_split_calls(ctx, variant, iters, monkeypatch):
    """PCG iterate after k iterations matches the oracle's (Saad) iterate for
    both variants, and k iterations split over several ebb_cg_step calls
    (scalars and buffer parity carried on the device) give the same iterate."""
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    case = Case(n=5, model="nh", vel_amp=0.05)
    fem = gpu_fem(ctx, case, name=f"cgit{variant}{iters}")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    out = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], 1e-2, iters=iters)
    fem.map_forces("nh")
    fem.assemble(1e-2)
    fem.cg_init()
    fem.cg_step(iters)
    x1 = fem.dv.read()
    assert rel_l2(x1, out["dv"]) <= 1e-9
    fem.cg_init()
    done = 0
    for k in (1, 2, 3, 100):
        k = min(k, iters - done)
        if k <= 0:
            break
        fem.cg_step(k)
        done += k
    # variant 3 sums the transposed blocks with red.add: run-to-run round-off
    assert rel_l2(fem.dv.read(), x1) <= (1e-13 if variant != "3" else 1e-11)
    assert ctx.error_counts(reset=True)["not_spd"] == 0


@pytest.mark.parametrize("variant,fallback", [("1", False), ("2", False), ("3", False), ("1", True)])
def test_cg_tolerance_mode(ctx, variant, fallback, monkeypatch):
    """SURVEY §8(f) 1, tolerance-based PCG: with ebb_cg.tol > 0 the solve stops
    on the device after the first iteration k with r_k.z_k <= tol^2 r_0.z_0.
    k is read off the oracle's r.z history on the same system (the stop rule
    is that definition), the iterate must be the oracle's k-th, later calls
    are no-ops, and tol = 0 keeps the fixed-iteration parity mode."""
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    if fallback:
        monkeypatch.setenv("EBB_CG", "2")            # one launch per phase (Saad)
    case = Case(n=6, model="nh", vel_amp=0.05)
    fem = gpu_fem(ctx, case, name=f"cgtol{variant}{int(fallback)}")
    fem.map_forces("nh")
    fem.assemble(1e-2)
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    free = case.free[order]
    # the oracle's own system of this step (its map and assembly; no GPU value)
    sysref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                                  free, 1e-2, iters=1)
    A, b = sysref["A"], sysref["b"]
    nmax = 400
    _, hist, _ = oracle.pcg(m.row_ptr, m.head, A, b, free, nmax)
    for tol in (1e-2, 1e-4):
        thr = tol * tol * hist[0]
        k = next(k for k in range(1, nmax + 1) if hist[k] <= thr)
        # fp64 decides the stop on both sides: the rule must not sit on the threshold
        assert abs(hist[k] - thr) > 1e-6 * thr and abs(hist[k - 1] - thr) > 1e-6 * thr
        x_ref, _, _ = oracle.pcg(m.row_ptr, m.head, A, b, free, k)
        fem.cg_init(tol=tol)
        fem.cg_step(3)
        fem.cg_step(nmax)
        assert fem.cg_iterations() == (k, True)
        x = fem.dv.read()
        assert rel_l2(x, x_ref) <= 1e-9
        fem.cg_step(10)                                  # converged: a no-op
        assert fem.cg_iterations() == (k, True)
        assert np.array_equal(fem.dv.read(), x)
    fem.cg_init(tol=0.0)
    fem.cg_step(4)
    fem.cg_step(3)
    assert fem.cg_iterations() == (7, False)
    x_ref, _, _ = oracle.pcg(m.row_ptr, m.head, A, b, free, 7)
    assert rel_l2(fem.dv.read(), x_ref) <= 1e-9
    assert ctx.error_counts(reset=True)["not_spd"] == 0


def test_consistent_mass_field(ctx):
    """ebb_tetmesh_consistent_mass against the oracle's Galerkin edge mass
    (fp64 atomics: equal up to summation order)."""
    case = Case(n=6, rho=850.0)
    fem = gpu_fem(ctx, case, name="cmass", mass="consistent")
    m, *_ = oracle_renumbered(case)
    ref = oracle.consistent_mass(m.e, m.W, 850.0, m.ne)
    got = fem.mass_e.read().ravel()
    assert np.abs(got - ref).max() <= 1e-14 * ref.max()
    assert np.all(got > 0)


@pytest.mark.parametrize("variant", ["1", "2"])
@pytest.mark.parametrize("model", ["nh", "stvk"])
def test_implicit_step_consistent_mass(ctx, model, variant, monkeypatch):
    """the implicit step with the consistent edge mass
    (A = M_c + hD + h^2 K, M v and M g as edge query-loops) reproduces the
    oracle's step, same bars as the lumped step."""
    monkeypatch.setenv("EBB_CG_VARIANT", variant)
    case = Case(n=6, model=model, vel_amp=0.05)
    h, iters, al, be = 1e-2, 50, 0.05, 0.002
    fem = gpu_fem(ctx, case, name=f"impc{model}{variant}", mass="consistent")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    out = oracle.implicit_step(m, model, case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], h, iters=iters, alpha=al, beta=be, mass="consistent")
    fem.implicit_step(model, h=h, iters=iters, alpha=al, beta=be)
    assert rel_l2(fem.b.read(), out["b"]) <= 1e-12
    assert rel_l2(fem.K.read(), out["A"]) <= 1e-12
    assert rel_l2(fem.dv.read(), out["dv"]) <= 1e-8
    assert rel_l2(fem.u.read(), out["u"]) <= 1e-8
    assert ctx.error_counts(reset=True)["not_spd"] == 0


@pytest.mark.parametrize("mass,model,newton", [("lumped", "nh", 3), ("consistent", "nh", 2), ("lumped", "stvk", 2)])
def test_implicit_newton_iterations(ctx, mass, model, newton, monkeypatch):
    """SURVEY §8(f) 1, several Newton iterations per backward-Euler step: the
    first is the one-linearisation step, each later one maps at
    u = u_n + h w, assembles b = h(f + Mg - Dw) + M(v_n - w) and updates
    w += dw, u += h dw -- against oracle.newton_step (bar 1e-8 on u, v; the
    later increments are small residual corrections, compared at 1e-6)."""
    monkeypatch.setenv("EBB_CG_VARIANT", "1")
    case = Case(n=6, model=model, vel_amp=0.05)
    h, iters, al, be = 1e-2, 50, 0.05, 0.002
    fem = gpu_fem(ctx, case, name=f"newt{mass}{model}{newton}", mass=mass)
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    out = oracle.newton_step(m, model, case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                             case.free[order], h, iters=iters, newton=newton, alpha=al, beta=be, mass=mass)
    fem.implicit_step(model, h=h, iters=iters, alpha=al, beta=be, newton=newton)
    assert rel_l2(fem.u.read(), out["u"]) <= 1e-8
    assert rel_l2(fem.vel.read(), out["v"]) <= 1e-8
    assert rel_l2(fem.b.read(), out["b"]) <= 1e-6
    assert rel_l2(fem.dv.read(), out["dv"]) <= 1e-6
    assert ctx.error_counts(reset=True)["not_spd"] == 0
