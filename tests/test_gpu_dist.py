"""Multi-GPU decomposition exercised on one B200 with virtual
ranks: every rank is a separate local problem (own relations, own CG state)
driven by the same distributed step as the torchrun path, with the
LocalTransport moving halo rows and scalar sums between them.  The owned
rows must reproduce the single-domain oracle implicit step."""
import numpy as np
import pytest

import oracle
from helpers import Case, oracle_renumbered, rel_l2

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


def _ranks(ctx, case, P, name, map_variant="overlap"):
    """P virtual ranks, each from its own device partition (ebb_partition_local)."""
    from paper_1506_07577_b200 import dist
    ranks = []
    for r in range(P):
        part = dist.partition_rank(ctx, case.X, case.tets, P, r, name=f"{name}p{r}")
        ranks.append(dist.GpuRank(ctx, r, part, case.X, case.free, case.u, case.vel, case.mu, case.lam,
                                  name=f"{name}r{r}", map_variant=map_variant, nranks=P))
    return ranks


@pytest.mark.parametrize("variant", ["saad", "single"])
@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_virtual_ranks_reproduce_single_domain(ctx, P, variant):
    """Both distributed PCG drivers (Saad: two allreduces per iteration;
    single-reduction phase mode: one fused allreduce and the u halo,
    SURVEY §8(e)) reproduce the single-domain oracle after 50 iterations."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, iters = 1e-2, 50
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], h, iters=iters)
    ranks = _ranks(ctx, case, P, f"v{P}{variant}")
    dist.implicit_step(ranks, dist.LocalTransport(), "nh", h=h, iters=iters, variant=variant)
    dv = np.full((m.nv, 3), np.nan)
    u = np.full((m.nv, 3), np.nan)
    for R in ranks:
        ids, vals = R.owned_values(R.fem.dv)
        dv[ids] = vals
        ids, vals = R.owned_values(R.fem.u)
        u[ids] = vals
    assert not np.isnan(dv).any()                 # every vertex owned exactly once
    assert rel_l2(dv[order], ref["dv"]) <= 1e-8
    assert rel_l2(u[order], ref["u"]) <= 1e-8


@pytest.mark.parametrize("map_variant", ["overlap", "reverse"])
@pytest.mark.parametrize("variant", ["saad", "single"])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_virtual_ranks_three_steps_owned_and_ghost_rows(ctx, P, variant, map_variant):
    """Three consecutive distributed implicit steps (50 PCG iterations each)
    match three single-domain oracle steps on EVERY local row, owned and
    ghost: step k+1 maps the ghost tets with the ghost u left by step k, so
    a stale ghost (the round-1 single-reduction driver left ghost dv at 0)
    corrupts the owned forces from step 2 on.  map_variant="reverse": every
    tet is mapped by one rank only and the partial f / K rows of ghost tails
    are added into their owners (the north_star halo of partial sums)."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, iters, steps = 1e-2, 50, 3
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    u, v = case.u[order], case.vel[order]
    for _ in range(steps):
        ref = oracle.implicit_step(m, "nh", u, v, case.mu[tet_src], case.lam[tet_src], case.free[order], h,
                                   iters=iters)
        u, v = ref["u"], ref["v"]
    ranks = _ranks(ctx, case, P, f"v3{P}{variant}{map_variant}", map_variant)
    u_in, v_in = np.empty_like(u), np.empty_like(v)
    u_in[order], v_in[order] = u, v                  # oracle (stored order) -> input rows
    u, v = u_in, v_in
    for _ in range(steps):
        dist.implicit_step(ranks, dist.LocalTransport(), "nh", h=h, iters=iters, variant=variant)
    nghost = 0
    for R in ranks:
        ids, gu = R.local_values(R.fem.u)
        _, gv = R.local_values(R.fem.vel)
        nghost += int((~R.owned_stored).sum())
        assert rel_l2(gu, u[ids]) <= 1e-8
        assert rel_l2(gv, v[ids]) <= 1e-8
        ghost = ~R.owned_stored
        assert rel_l2(gu[ghost], u[ids[ghost]]) <= 1e-8
        assert rel_l2(gv[ghost], v[ids[ghost]]) <= 1e-8
    assert nghost > 0


@pytest.mark.parametrize("mode", ["overlap", "own"])
@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_partition_local_matches_oracle(ctx, P, mode):
    """ebb_partition_local (device) == oracle O4 bit-exact for every rank:
    local tets, local vertices (owned then ghosts), the local tet keys and
    every send / recv list; the global relations are freed afterwards."""
    from paper_1506_07577_b200 import dist
    case = Case(n=5, model="nh")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.partition(m.nv, m.tets, P, mode=mode)
    for r in range(P):
        part = dist.partition_rank(ctx, case.X, case.tets, P, r, name=f"pl{P}{mode}{r}", mode=mode, debug=True)
        assert np.array_equal(part["vert_order"], order)              # device renumbering == O3
        assert np.array_equal(part["owner_v"], ref["owner_v"])          # device owner map == O4
        st_v = np.empty_like(order)
        st_v[order] = np.arange(order.size)                            # input row -> stored id
        st_t = np.empty_like(part["tet_order"])
        st_t[part["tet_order"]] = np.arange(st_t.size)
        lv = st_v[part["vert_src"]]
        assert np.array_equal(lv, ref["local"][r])
        assert part["n_owned"] == int((ref["owner_v"] == r).sum())
        assert np.array_equal(st_t[part["tet_src"]], ref["ltets"][r])
        assert np.array_equal(lv[part["tets"]], m.tets[ref["ltets"][r]])
        for q in range(P):
            s_rows = part["send"].get(q, np.zeros(0, np.int64))
            r_rows = part["recv"].get(q, np.zeros(0, np.int64))
            assert np.array_equal(lv[s_rows], ref["send"][r][q])
            assert np.array_equal(lv[r_rows], ref["send"][q][r])


def test_relation_and_field_free(ctx):
    """ebb_relation_free / ebb_field_free: handles become invalid, a relation
    still targeted by another relation's key-field is refused, names are
    reusable after the free."""
    from paper_1506_07577_b200.ebb import EbbError
    A_ = ctx.relation("freeA", 10)
    B_ = ctx.relation("freeB", 4)
    x = A_.field("x", "f64", init=np.arange(10.0))
    k = B_.key_field("k", A_, (1, 1), np.array([0, 3, 5, 9], dtype=np.uint64))
    with pytest.raises(EbbError, match="EBB_E_STATE"):
        A_.free()                                   # B.k targets A
    x.free()
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        x.read()
    B_.free()
    A_.free()
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        k.read()
    A2 = ctx.relation("freeA", 3)                   # the name is free again
    assert A2.field("y", "f64", init=np.ones(3)).read().tolist() == [1.0, 1.0, 1.0]


@pytest.mark.parametrize("variant", ["saad", "single"])
def test_nccl_transport_single_rank(ctx, variant):
    """The in-library NCCL transport (ebb_comm_*; a 1-rank communicator on
    this one-GPU box) drives the distributed step to the oracle's result: the
    allreduces of the PCG scalars and the (empty) halo go through NCCL."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, iters = 1e-2, 50
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], h, iters=iters)
    (R,) = _ranks(ctx, case, 1, f"nccl1{variant}")
    T = dist.NcclTransport(ctx, 0, 1)
    dist.implicit_step([R], T, "nh", h=h, iters=iters, variant=variant)
    ids, dv = R.owned_values(R.fem.dv)
    out = np.full((m.nv, 3), np.nan)
    out[ids] = dv
    assert rel_l2(out[order], ref["dv"]) <= 1e-8


def test_nccl_allreduce_and_errors(ctx):
    """ebb_comm_allreduce_sum on a device buffer (1 rank: identity) and the
    state error before ebb_comm_init on a fresh context."""
    import ctypes as C

    import torch

    from paper_1506_07577_b200 import dist, ebb
    fresh = ebb.Context(0)
    buf = torch.arange(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ebb.EbbError, match="EBB_E_STATE"):
        fresh.check(fresh.L.ebb_comm_allreduce_sum(fresh.h, buf.data_ptr(), 4, None))
    dist.NcclTransport(fresh, 0, 1)
    fresh.check(fresh.L.ebb_comm_allreduce_sum(fresh.h, buf.data_ptr(), 4, None))
    torch.cuda.synchronize()
    assert buf.tolist() == [0.0, 1.0, 2.0, 3.0]
    fresh.close()
    del C


def test_single_reduction_phases_honour_the_tolerance(ctx):
    """Phase mode with ebb_cg.tol > 0 on 2 virtual ranks: the solve stops on
    the device at the oracle's stop iteration (read off its r.z history of the
    single-domain system) and later phases are no-ops."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, P, tol = 1e-2, 2, 1e-3
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], h, iters=1)
    _, hist, _ = oracle.pcg(m.row_ptr, m.head, ref["A"], ref["b"], case.free[order], 300)
    thr = tol * tol * hist[0]
    k = next(k for k in range(1, 301) if hist[k] <= thr)
    assert abs(hist[k] - thr) > 1e-6 * thr and abs(hist[k - 1] - thr) > 1e-6 * thr
    x_ref, _, _ = oracle.pcg(m.row_ptr, m.head, ref["A"], ref["b"], case.free[order], k)
    ranks = _ranks(ctx, case, P, "vtol")
    for R in ranks:
        R.fem.cg.tol = tol
    dist.implicit_step(ranks, dist.LocalTransport(), "nh", h=h, iters=k + 40, variant="single")
    dv = np.full((m.nv, 3), np.nan)
    for R in ranks:
        ids, vals = R.owned_values(R.fem.dv)
        dv[ids] = vals
        assert R.fem.cg_iterations() == (k, True)
    assert rel_l2(dv[order], x_ref) <= 1e-8


@pytest.mark.parametrize("P", [2, 4])
def test_reverse_add_maps_every_tet_once(ctx, P):
    """The reverse-add variant maps each tet on exactly one rank (the tets the
    ranks map partition the mesh), and one distributed step equals the
    single-domain oracle; the overlap variant maps more tets in total."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ranks = _ranks(ctx, case, P, f"rv1{P}", "reverse")
    assert sum(R.n_map_tets for R in ranks) == m.nt
    assert sum(R.fem.nt for R in ranks) > m.nt                       # the overlap's ghost tets
    assert all(R.rev_bytes["rK"] > 0 for R in ranks)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], 1e-2, iters=50)
    dist.implicit_step(ranks, dist.LocalTransport(), "nh", h=1e-2, iters=50, variant="single")
    dv = np.full((m.nv, 3), np.nan)
    for R in ranks:
        ids, vals = R.owned_values(R.fem.dv)
        dv[ids] = vals
    assert rel_l2(dv[order], ref["dv"]) <= 1e-8


@pytest.mark.parametrize("halo", ["transport", "peer"])
@pytest.mark.parametrize("map_variant", ["overlap", "reverse"])
@pytest.mark.parametrize("model,dtype", [("stvk", "f64"), ("nh", "f64"), ("stvk", "f32")])
@pytest.mark.parametrize("P", [2, 3])
def test_distributed_map_step(ctx, P, model, dtype, map_variant, halo):
    """BASELINE configs[2]'s distributed map: after the position halo and the
    map (plus the reverse add), every owned force row and every owned
    stiffness row equals the single-domain oracle's: f directly, K through
    K p for a seeded global p (each owned row of K p uses the whole row).
    The ranks start from stale ghost displacements (zeros), so the halo
    exchange is what makes the ghost tets right.  halo="peer": the position
    halo as the peer-memory push kernel (ebb_peer_halo_push, COPY) and, for
    the reverse variant, the partial f / K rows added into their owners with
    red.global.add over peer memory (ADD) -- no transport at all; the ranks
    emulated in one cooperative launch."""
    from paper_1506_07577_b200 import dist
    case = Case(n=5, model=model, spread=0.1)
    if dtype == "f32":
        for k in ("u", "mu", "lam"):
            setattr(case, k, getattr(case, k).astype(np.float32).astype(np.float64))
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    f, K, en, inv = oracle.element_map(model, m.X, case.u[order], m.tets, m.Dminv, m.W, case.mu[tet_src],
                                       case.lam[tet_src], e=m.e, ne=m.ne)
    rng = np.random.default_rng(9)
    p_in = rng.uniform(-1, 1, size=(m.nv, 3))                  # input order
    Kp = oracle.edge_matvec(m.row_ptr, m.head, K, p_in[order])  # stored order
    ranks = []
    for r in range(P):
        part = dist.partition_rank(ctx, case.X, case.tets, P, r, name=f"dm{P}{model}{dtype}{map_variant}{halo}p{r}")
        u_stale = case.u.copy()
        R = dist.GpuRank(ctx, r, part, case.X, case.free, u_stale, case.vel, case.mu, case.lam, dtype=dtype,
                         name=f"dm{P}{model}{dtype}{map_variant}{halo}r{r}", map_variant=map_variant, nranks=P)
        ghost = ~R.owned_stored
        uu = R.fem.u.read()
        uu[ghost] = 0.0                                         # stale ghosts: the halo must refresh them
        R.fem.u.write(uu)
        ranks.append(R)
    ph = dist.PeerHalo(ranks) if halo == "peer" else None
    prev = (dist.PeerHalo(ranks, "rf"), dist.PeerHalo(ranks, "rK")) if halo == "peer" and map_variant == "reverse" \
        else None                                               # the reverse add as peer-memory REDs
    dist.map_step(ranks, None if halo == "peer" else dist.LocalTransport(), model, halo=ph, peer_rev=prev)
    assert ctx.error_counts()["peer_timeouts"] == 0
    tol = 1e-12 if dtype == "f64" else 1e-5
    f_in = np.full((m.nv, 3), np.nan)
    kp_in = np.full((m.nv, 3), np.nan)
    for R in ranks:
        ids, vals = R.owned_values(R.fem.f)
        f_in[ids] = vals
        Pf = R.fem.verts.field("p_dm", dtype, (3, 1), init=p_in[R.verts_g])
        Qf = R.fem.verts.field("q_dm", dtype, (3, 1))
        R.fem.matvec(R.fem.K, Pf, Qf)
        kp_in[ids] = Qf.read()[R.owned_stored]
    assert rel_l2(f_in[order], f) <= tol
    assert rel_l2(kp_in[order], Kp) <= tol


def test_partition_and_halo_entry_points_refuse_bad_arguments(ctx):
    """Argument checks of the round-2 multi-GPU entry points: a rank outside
    [0, nparts), an unknown mode, owner fields of the wrong type, a
    scatter-add into a key-field or an integer field, reverse lists from
    fields on the wrong relations."""
    import ctypes as C

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200.ebb import EbbError
    case = Case(n=3)
    V = ctx.relation("bad.verts", case.X.shape[0])
    T = ctx.relation("bad.tets", case.tets.shape[0])
    v = T.key_field("v", V, (4, 1), case.tets)
    ot, ov = T.field("ot", "i32"), V.field("ov", "i32")
    ctx.check(ctx.L.ebb_partition(ctx.h, v.h, 2, ot.h, ov.h))
    info = A.PartitionInfo()
    sp, rp = (C.c_uint64 * 3)(), (C.c_uint64 * 3)()
    for rank, mode, o_t, o_v, err in ((2, 0, ot, ov, "EBB_E_ARG"), (0, 7, ot, ov, "EBB_E_ARG"),
                                      (0, 0, ov, ot, "EBB_E_TYPE")):
        with pytest.raises(EbbError, match=err):
            ctx.check(ctx.L.ebb_partition_local(ctx.h, v.h, o_t.h, o_v.h, 2, rank, mode, b"bad", C.byref(info),
                                                sp, rp))
    rows = V.field("rows_b", "u32", init=np.arange(case.X.shape[0], dtype=np.uint32))
    buf = V.field("buf_b", "u32")
    with pytest.raises(EbbError):
        ctx.check(ctx.L.ebb_rows_scatter_add(ctx.h, v.h, rows.h, buf.h, None))     # key-field target
    ivals = V.field("ival", "i32")
    ibuf = V.field("ibuf", "i32")
    with pytest.raises(EbbError, match="EBB_E_TYPE"):
        ctx.check(ctx.L.ebb_rows_scatter_add(ctx.h, ivals.h, rows.h, ibuf.h, None))
    rinfo = A.ReverseInfo()
    ptr = (C.c_uint64 * 12)()
    with pytest.raises(EbbError, match="EBB_E_TYPE"):
        ctx.check(ctx.L.ebb_partition_reverse(ctx.h, v.h, v.h, rows.h, ov.h, 2, 0, b"badrev", C.byref(rinfo), ptr))


@pytest.mark.parametrize("P", [2, 3, 4])
def test_partition_reverse_matches_oracle(ctx, P):
    """ebb_partition_reverse (device) == oracle.partition_reverse bit-exact
    for every rank and peer, in global ids: the force rows sent and received
    (vertex ids) and the stiffness rows sent and received ((tail, head) of
    the local edge rows), each in the order both ends derive."""
    case = Case(n=5, model="nh")
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    # the key of the lowest-vertex rule and of the list order: the input row
    # of every (renumbered) vertex, as GpuRank passes it
    ref = oracle.partition_reverse(m.nv, m.tets, P, key=order)
    st_v = np.empty_like(order)
    st_v[order] = np.arange(order.size)                 # input row -> stored (global) id
    ranks = _ranks(ctx, case, P, f"prv{P}", "reverse")
    none = np.zeros(0, np.int64)
    for R in ranks:
        g = st_v[R.verts_g]                              # local vertex row -> global id
        index = R.fem.index.read().astype(np.int64)
        head = R.fem.head.read().astype(np.int64)
        tail = np.repeat(np.arange(R.fem.nv), np.diff(index))
        fsend, frecv = R.rev_lists["rf"]
        ksend, krecv = R.rev_lists["rK"]
        pairs = lambda rows: np.stack([g[tail[rows]], g[head[rows]]], axis=1) if len(rows) else \
            np.zeros((0, 2), np.int64)                  # noqa: E731
        for q in range(P):
            if q == R.rank:
                continue
            assert np.array_equal(g[np.asarray(fsend.get(q, none))], ref["fsend"][R.rank][q])
            assert np.array_equal(g[np.asarray(frecv.get(q, none))], ref["fsend"][q][R.rank])
            assert np.array_equal(pairs(np.asarray(ksend.get(q, none))), ref["ksend"][R.rank][q])
            assert np.array_equal(pairs(np.asarray(krecv.get(q, none))), ref["ksend"][q][R.rank])
