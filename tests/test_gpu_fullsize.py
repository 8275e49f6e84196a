"""Full-size parity at BASELINE configs[2] (C3): StVK / NH force+stiffness map
on the ~1e7-tet blob, fp32, in the launch configuration the sweep times.
The oracle cannot run the whole map in seconds, so it computes exact rows for
a seeded sample of vertices: the sub-mesh of every tet touching a sampled
vertex reproduces that vertex's force and all of its stiffness rows."""
import numpy as np
import pytest

import oracle
from helpers import rel_l2
from synth import mesh as M
from synth import state as S

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


@pytest.fixture(scope="module")
def c3():
    X, tets, n = M.blob(10_000_000)
    free = S.fixed_mask(X, n)
    u = S.twist_u(X, n, 6, free=free).astype(np.float32).astype(np.float64)
    mu, lam = S.materials(tets.shape[0], 1e6, 0.3, spread=0.1)
    mu = mu.astype(np.float32).astype(np.float64)
    lam = lam.astype(np.float32).astype(np.float64)
    new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
    return dict(X=X, tets=tets, n=n, free=free, u=u, mu=mu, lam=lam, new_of_old=new_of_old, tet_src=tet_src,
                tets_new=tets_new)


@pytest.mark.parametrize("model", ["stvk", "nh"])
def test_c3_blob_map_sampled_rows(ctx, c3, model):
    from paper_1506_07577_b200.tetfem import TetFEM
    d = c3
    fem = TetFEM(ctx, d["X"], d["tets"], dtype="f32", mu=d["mu"], lam=d["lam"], free=d["free"], u=d["u"],
                 name=f"c3{model}")
    order = np.argsort(d["new_of_old"])
    assert np.array_equal(fem.vert_order(), order)            # a2 bit-exact at 1e7 tets
    assert np.array_equal(fem.tet_order(), d["tet_src"])
    fem.map_forces(model)
    f_gpu = fem.f.read()
    index = fem.index.read().astype(np.int64)
    head = fem.head.read().astype(np.int64)
    K_gpu = fem.K.read().reshape(-1, 3, 3)
    # seeded vertex sample, all their incident tets (stored numbering)
    Xs = d["X"][order]
    tets_s = d["tets_new"]
    rng = M.rng(11)
    sample = np.unique(rng.integers(0, Xs.shape[0], size=400))
    touch = np.isin(tets_s, sample).any(axis=1)
    sub_t = np.nonzero(touch)[0]
    sub_v = np.unique(tets_s[sub_t])
    local = np.searchsorted(sub_v, tets_s[sub_t])
    m = oracle.Mesh(Xs[sub_v], local)
    mu_s, lam_s = d["mu"][d["tet_src"]][sub_t], d["lam"][d["tet_src"]][sub_t]
    f, K, en, inv = oracle.element_map(model, m.X, d["u"][order][sub_v], m.tets, m.Dminv, m.W, mu_s, lam_s,
                                       e=m.e, ne=m.ne)
    li = np.searchsorted(sub_v, sample)
    assert rel_l2(f_gpu[sample], f[li]) <= 1e-5
    got, ref = [], []
    for v, lv in zip(sample, li):
        heads_gpu = head[index[v]:index[v + 1]]
        heads_ora = sub_v[m.head[m.row_ptr[lv]:m.row_ptr[lv + 1]]]
        assert np.array_equal(heads_gpu, heads_ora)           # same edge rows, same order
        got.append(K_gpu[index[v]:index[v + 1]])
        ref.append(K[m.row_ptr[lv]:m.row_ptr[lv + 1]])
    assert rel_l2(np.concatenate(got), np.concatenate(ref)) <= 1e-5


@pytest.fixture(scope="module")
def t10m():
    """bench.py's workload (T10M: Kuhn-6 n=119, 10,110,954 tets, the
    wall-ramped stretch recipe, E scaled for n) and the oracle's O3 order."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench
    w = bench.WORKLOAD
    X, tets, free, u, mu, lam = bench.make_case(w["n"], w["order_seed"], w["u_seed"], w["E"], w["nu"],
                                                wall_ramp=w["wall_ramp"])
    new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
    return dict(w=w, X=X, tets=tets, free=free, u=u, mu=mu, lam=lam, new_of_old=new_of_old, tet_src=tet_src,
                tets_new=tets_new)


def test_t10m_map_and_assembly_sampled_rows(ctx, t10m):
    """Full-size parity at the bench's own configuration (fp64 NH, the
    SEGMENTED map with its device-built plan, the fused assembly), on a seeded
    sample of vertices the oracle computes exactly from the sub-mesh of their
    incident tets: renumbering bit-exact, forces, every stiffness row, every
    system row A = M + h^2 K and the right-hand side b of the sample <= 1e-12."""
    from paper_1506_07577_b200.tetfem import TetFEM
    d = t10m
    w = d["w"]
    fem = TetFEM(ctx, d["X"], d["tets"], dtype="f64", mu=d["mu"], lam=d["lam"], rho=w["rho"], free=d["free"],
                 u=d["u"], name="t10m")
    order = np.argsort(d["new_of_old"])
    assert np.array_equal(fem.vert_order(), order)            # a2 bit-exact at 1e7 tets
    assert np.array_equal(fem.tet_order(), d["tet_src"])
    fem.map_forces(w["model"])
    f_gpu = fem.f.read()
    K_gpu = fem.K.read().reshape(-1, 9)
    fem.assemble(w["h"])
    A_gpu = fem.K.read().reshape(-1, 9)                         # A overwrites K in place (a9)
    b_gpu = fem.b.read()
    index = fem.index.read().astype(np.int64)
    head = fem.head.read().astype(np.int64)
    Xs, tets_s = d["X"][order], d["tets_new"]
    rng = M.rng(12)
    sample = np.unique(rng.integers(0, Xs.shape[0], size=300))
    sub_t = np.nonzero(np.isin(tets_s, sample).any(axis=1))[0]
    sub_v = np.unique(tets_s[sub_t])
    m = oracle.Mesh(Xs[sub_v], np.searchsorted(sub_v, tets_s[sub_t]), rho=w["rho"])
    f, K, en, inv = oracle.element_map(w["model"], m.X, d["u"][order][sub_v], m.tets, m.Dminv, m.W,
                                       d["mu"][d["tet_src"]][sub_t], d["lam"][d["tet_src"]][sub_t], e=m.e, ne=m.ne)
    A, b = oracle.implicit_assemble(m.row_ptr, m.head, K, m.mass, f, np.zeros((m.nv, 3)), w["h"])
    li = np.searchsorted(sub_v, sample)
    assert rel_l2(f_gpu[sample], f[li]) <= 1e-12
    assert rel_l2(b_gpu[sample], b[li]) <= 1e-12
    gk, rk, ga, ra = [], [], [], []
    for v, lv in zip(sample, li):
        assert np.array_equal(head[index[v]:index[v + 1]], sub_v[m.head[m.row_ptr[lv]:m.row_ptr[lv + 1]]])
        gk.append(K_gpu[index[v]:index[v + 1]])
        rk.append(K[m.row_ptr[lv]:m.row_ptr[lv + 1]].reshape(-1, 9))
        ga.append(A_gpu[index[v]:index[v + 1]])
        ra.append(A[m.row_ptr[lv]:m.row_ptr[lv + 1]].reshape(-1, 9))
    assert rel_l2(np.concatenate(gk), np.concatenate(rk)) <= 1e-12
    assert rel_l2(np.concatenate(ga), np.concatenate(ra)) <= 1e-12


def test_t10m_pcg_residual_property(ctx, t10m):
    """The bench's 50-iteration PCG at full size (Saad, one persistent launch):
    a property that holds at any size -- the recurrence residual r_50 the
    kernel carries equals the true residual b - A x_50, which the host
    recomputes in fp64 from the assembled rows on a seeded sample of free
    vertices (independent arithmetic) -- and the solve made progress
    (||r_50|| well below ||r_0|| = ||b|| on the free rows)."""
    from paper_1506_07577_b200 import _abi as A_
    from paper_1506_07577_b200.ebb import Field
    from paper_1506_07577_b200.tetfem import TetFEM
    d = t10m
    w = d["w"]
    fem = TetFEM(ctx, d["X"], d["tets"], dtype="f64", mu=d["mu"], lam=d["lam"], rho=w["rho"], free=d["free"],
                 u=d["u"], name="t10mcg")
    fem.map_forces(w["model"])
    fem.assemble(w["h"])
    fem.cg_init()
    assert fem.cg_variant() == A_.CG_SAAD
    fem.cg_step(w["cg_iters"])
    x = fem.dv.read()
    r = Field(ctx, fem.cg.r, fem.verts, "r", "f64", (4, 1), A_.AOS).read()[:, :3]
    b = fem.b.read()
    Arows = fem.K.read().reshape(-1, 3, 3)
    index = fem.index.read().astype(np.int64)
    head = fem.head.read().astype(np.int64)
    free = fem.free.read().astype(bool)
    rng = M.rng(13)
    sample = np.unique(rng.integers(0, fem.nv, size=2000))
    sample = sample[free[sample]]
    rt = np.empty((sample.size, 3))
    for k, v in enumerate(sample):
        e0, e1 = index[v], index[v + 1]
        rt[k] = b[v] - np.einsum("eab,eb->a", Arows[e0:e1], x[head[e0:e1]])
    assert rel_l2(r[sample], rt) <= 1e-8
    assert np.linalg.norm(r[free]) < 1e-2 * np.linalg.norm(b[free])


@pytest.mark.parametrize("body", ["saad", "single"])
def test_t10m_peer_pcg_two_ranks(ctx, t10m, body):
    """The fused multi-GPU PCG (bench.py --gpus N's default; both kernel
    bodies) at full size: the T10M mesh split over 2 ranks emulated on the
    GPU (one cooperative launch).  Properties that hold at any size, per rank
    on a seeded sample of owned free rows that includes every boundary row
    of the sample's range: the recurrence residual equals b - A x computed on
    the host from the local rows and the local x -- whose ghost rows the
    peer stored into this rank inside the kernel -- and the distributed
    step's dv and u, owned and ghost rows, equal the single-domain step's
    (the same iterates in exact arithmetic; north_star's 1e-8 CG bar)."""
    from paper_1506_07577_b200 import _abi as A_
    from paper_1506_07577_b200 import dist
    from paper_1506_07577_b200.ebb import Field
    from paper_1506_07577_b200.tetfem import TetFEM
    d = t10m
    w = d["w"]
    v0 = np.zeros_like(d["u"])
    ranks = []
    for r in range(2):
        part = dist.partition_rank(ctx, d["X"], d["tets"], 2, r, name=f"t10mpp{body}{r}")
        ranks.append(dist.GpuRank(ctx, r, part, d["X"], d["free"], d["u"], v0, d["mu"], d["lam"], rho=w["rho"],
                                  name=f"t10mpr{body}{r}", nranks=2))
    peer = dist.PeerPCG(ranks, variant=body)
    dist.implicit_step(ranks, None, w["model"], h=w["h"], iters=w["cg_iters"], variant="peer", peer=peer)
    assert ctx.error_counts()["peer_timeouts"] == 0
    rng = M.rng(14)
    for R in ranks:
        f = R.fem
        x = f.dv.read()
        rr = Field(ctx, f.cg.r, f.verts, "r", "f64", (4, 1), A_.AOS).read()[:, :3]
        b = f.b.read()
        Arows = f.K.read().reshape(-1, 3, 3)
        index = f.index.read().astype(np.int64)
        head = f.head.read().astype(np.int64)
        free = f.free.read().astype(bool)                       # mask = free AND owned
        bnd = np.unique(np.concatenate([np.asarray(s) for s in R.part_send.values()]))
        sample = np.unique(np.concatenate([rng.integers(0, R.n_owned, size=1000), bnd[:1000]]))
        sample = sample[free[sample]]
        assert np.isin(bnd, sample).sum() > 100                 # rows whose A x reads ghost x
        rt = np.empty((sample.size, 3))
        for k, v in enumerate(sample):
            e0, e1 = index[v], index[v + 1]
            rt[k] = b[v] - np.einsum("eab,eb->a", Arows[e0:e1], x[head[e0:e1]])
        assert rel_l2(rr[sample], rt) <= 1e-8
    # the single-domain step on the same input (bench.py's single-GPU path)
    fem = TetFEM(ctx, d["X"], d["tets"], dtype="f64", mu=d["mu"], lam=d["lam"], rho=w["rho"], free=d["free"],
                 u=d["u"], name=f"t10mref{body}")
    fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"])
    dv_ref = fem.to_input_order(fem.dv.read())
    u_ref = fem.to_input_order(fem.u.read())
    dv = np.full_like(dv_ref, np.nan)
    u = np.full_like(u_ref, np.nan)
    for R in ranks:
        ids, vals = R.local_values(R.fem.dv)                     # owned and ghost rows
        dv[ids] = vals
        ids, vals = R.local_values(R.fem.u)
        u[ids] = vals
    assert not np.isnan(dv).any()
    assert rel_l2(dv, dv_ref) <= 1e-8                           # north_star's CG-iterate bar
    assert rel_l2(u, u_ref) <= 1e-8


def test_t10m_transport_free_reverse_add_step(ctx, t10m):
    """The whole transport-free distributed step at full size with north_star's
    reverse add: T10M over 2 emulated ranks, each tet mapped once, the
    partial f / K rows of ghost tails added into their owners with
    red.global.add over peer memory (PeerHalo ADD), the fused peer PCG
    (Saad body): dv and u on every local row equal the single-domain step's
    (north_star's 1e-8 CG bar)."""
    from paper_1506_07577_b200 import dist
    from paper_1506_07577_b200.tetfem import TetFEM
    d = t10m
    w = d["w"]
    v0 = np.zeros_like(d["u"])
    ranks = []
    for r in range(2):
        part = dist.partition_rank(ctx, d["X"], d["tets"], 2, r, name=f"t10mrv{r}")
        ranks.append(dist.GpuRank(ctx, r, part, d["X"], d["free"], d["u"], v0, d["mu"], d["lam"], rho=w["rho"],
                                  name=f"t10mrvr{r}", map_variant="reverse", nranks=2))
    assert sum(R.n_map_tets for R in ranks) == d["tets"].shape[0]     # every tet mapped once
    peer = dist.PeerPCG(ranks, variant="saad")
    prev = (dist.PeerHalo(ranks, "rf"), dist.PeerHalo(ranks, "rK"))
    dist.implicit_step(ranks, None, w["model"], h=w["h"], iters=w["cg_iters"], variant="peer", peer=peer,
                       peer_rev=prev)
    assert ctx.error_counts()["peer_timeouts"] == 0
    fem = TetFEM(ctx, d["X"], d["tets"], dtype="f64", mu=d["mu"], lam=d["lam"], rho=w["rho"], free=d["free"],
                 u=d["u"], name="t10mrvref")
    fem.implicit_step(w["model"], h=w["h"], iters=w["cg_iters"])
    dv_ref = fem.to_input_order(fem.dv.read())
    u_ref = fem.to_input_order(fem.u.read())
    for R in ranks:
        ids, dv = R.local_values(R.fem.dv)
        _, u = R.local_values(R.fem.u)
        assert rel_l2(dv, dv_ref[ids]) <= 1e-8
        assert rel_l2(u, u_ref[ids]) <= 1e-8
