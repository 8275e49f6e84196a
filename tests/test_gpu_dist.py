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
    G = dist.global_partition(ctx, case.X, case.tets, P, name=f"vg{P}{variant}")
    assert np.array_equal(G["vert_order"], order)            # device renumbering == oracle O3
    ref_part = oracle.partition(m.nv, m.tets, P)
    assert np.array_equal(G["owner_v"], ref_part["owner_v"])  # device O4 == oracle O4
    plan = dist.halo_plan(G["tets"], G["owner_v"], P)
    tord = G["tet_order"]
    ranks = [dist.GpuRank(ctx, r, G["X"], G["tets"], G["owner_v"], plan, case.free[order], case.u[order],
                          case.vel[order], case.mu[tord], case.lam[tord], name=f"v{P}{variant}r{r}")
             for r in range(P)]
    dist.implicit_step(ranks, dist.LocalTransport(), "nh", h=h, iters=iters, variant=variant)
    dv = np.full((m.nv, 3), np.nan)
    u = np.full((m.nv, 3), np.nan)
    for R in ranks:
        ids, vals = R.owned_values(R.fem.dv)
        dv[ids] = vals
        ids, vals = R.owned_values(R.fem.u)
        u[ids] = vals
    assert not np.isnan(dv).any()                 # every vertex owned exactly once
    assert rel_l2(dv, ref["dv"]) <= 1e-8
    assert rel_l2(u, ref["u"]) <= 1e-8


@pytest.mark.parametrize("variant", ["saad", "single"])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_virtual_ranks_three_steps_owned_and_ghost_rows(ctx, P, variant):
    """Three consecutive distributed implicit steps (50 PCG iterations each)
    match three single-domain oracle steps on EVERY local row, owned and
    ghost: step k+1 maps the ghost tets with the ghost u left by step k, so
    a stale ghost (the round-1 single-reduction driver left ghost dv at 0)
    corrupts the owned forces from step 2 on."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, iters, steps = 1e-2, 50, 3
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    u, v = case.u[order], case.vel[order]
    for _ in range(steps):
        ref = oracle.implicit_step(m, "nh", u, v, case.mu[tet_src], case.lam[tet_src], case.free[order], h,
                                   iters=iters)
        u, v = ref["u"], ref["v"]
    G = dist.global_partition(ctx, case.X, case.tets, P, name=f"v3g{P}{variant}")
    plan = dist.halo_plan(G["tets"], G["owner_v"], P)
    tord = G["tet_order"]
    ranks = [dist.GpuRank(ctx, r, G["X"], G["tets"], G["owner_v"], plan, case.free[order], case.u[order],
                          case.vel[order], case.mu[tord], case.lam[tord], name=f"v3{P}{variant}r{r}")
             for r in range(P)]
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


def test_halo_plan_is_consistent(ctx):
    from paper_1506_07577_b200 import dist
    case = Case(n=5)
    m, *_ = oracle_renumbered(case)
    part = oracle.partition(m.nv, m.tets, 3)
    problems, send, recv = dist.halo_plan(m.tets, part["owner_v"], 3)
    for r in range(3):
        lt, verts, ltets, owned = problems[r]
        # owner-computes: every tet touching an owned vertex is local
        touching = np.nonzero((part["owner_v"][m.tets] == r).any(axis=1))[0]
        assert np.array_equal(lt, touching)
        assert np.array_equal(np.sort(np.concatenate([recv[r][o] for o in range(3)])), verts[~owned])
        for o in range(3):
            assert np.array_equal(send[o][r], recv[r][o])
            assert np.all(part["owner_v"][send[o][r]] == o)


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
    G = dist.global_partition(ctx, case.X, case.tets, 1, name=f"nccl1{variant}")
    plan = dist.halo_plan(G["tets"], G["owner_v"], 1)
    tord = G["tet_order"]
    R = dist.GpuRank(ctx, 0, G["X"], G["tets"], G["owner_v"], plan, case.free[order], case.u[order],
                     case.vel[order], case.mu[tord], case.lam[tord], name=f"nccl1{variant}r0")
    T = dist.NcclTransport(ctx, 0, 1)
    dist.implicit_step([R], T, "nh", h=h, iters=iters, variant=variant)
    ids, dv = R.owned_values(R.fem.dv)
    out = np.full((m.nv, 3), np.nan)
    out[ids] = dv
    assert rel_l2(out, ref["dv"]) <= 1e-8


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
    G = dist.global_partition(ctx, case.X, case.tets, P, name="vgtol")
    plan = dist.halo_plan(G["tets"], G["owner_v"], P)
    tord = G["tet_order"]
    ranks = [dist.GpuRank(ctx, r, G["X"], G["tets"], G["owner_v"], plan, case.free[order], case.u[order],
                          case.vel[order], case.mu[tord], case.lam[tord], name=f"vtol{r}") for r in range(P)]
    for R in ranks:
        R.fem.cg.tol = tol
    dist.implicit_step(ranks, dist.LocalTransport(), "nh", h=h, iters=k + 40, variant="single")
    dv = np.full((m.nv, 3), np.nan)
    for R in ranks:
        ids, vals = R.owned_values(R.fem.dv)
        dv[ids] = vals
        assert R.fem.cg_iterations() == (k, True)
    assert rel_l2(dv, x_ref) <= 1e-8
