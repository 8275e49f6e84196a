"""The fused multi-GPU PCG over peer memory (ebb_cg_peer_bind / _step,
SURVEY §8(e)) on ranks emulated on one B200: every rank is its own local
problem (own relations, own CG state); one cooperative launch runs all of
them, the owners store u, x and z_0 into their peers' ghost rows and the
scalar sums go through the peers' mailboxes inside the kernel -- exactly the
kernel a one-process-per-GPU job launches with IPC-mapped peer buffers.
The results must reproduce the single-domain oracle (north_star: CG
iterates <= 1e-8 after 50 iterations), on owned AND ghost rows."""
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
    errs = c.error_counts()
    c.close()
    assert errs["peer_timeouts"] == 0, "a peer wait was abandoned"


def _ranks(ctx, case, P, name, map_variant="overlap", dtype="f64"):
    from paper_1506_07577_b200 import dist
    ranks = []
    for r in range(P):
        part = dist.partition_rank(ctx, case.X, case.tets, P, r, name=f"{name}p{r}")
        ranks.append(dist.GpuRank(ctx, r, part, case.X, case.free, case.u, case.vel, case.mu, case.lam,
                                  name=f"{name}r{r}", map_variant=map_variant, nranks=P, dtype=dtype))
    return ranks


def _gather(ranks, field, nv):
    out = np.full((nv, 3), np.nan)
    for R in ranks:
        ids, vals = R.owned_values(getattr(R.fem, field))
        out[ids] = vals
    return out


@pytest.mark.parametrize("variant", ["single", "saad"])
@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_peer_pcg_matches_single_domain(ctx, P, variant):
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, iters = 1e-2, 50
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], h, iters=iters)
    ranks = _ranks(ctx, case, P, f"pp{P}{variant}")
    peer = dist.PeerPCG(ranks, variant=variant)
    dist.implicit_step(ranks, None, "nh", h=h, iters=iters, variant="peer", peer=peer)
    dv = _gather(ranks, "dv", m.nv)
    u = _gather(ranks, "u", m.nv)
    assert not np.isnan(dv).any()
    assert rel_l2(dv[order], ref["dv"]) <= 1e-8
    assert rel_l2(u[order], ref["u"]) <= 1e-8
    for R in ranks:
        assert R.fem.cg_iterations()[0] == iters


@pytest.mark.parametrize("variant", ["single", "saad"])
@pytest.mark.parametrize("map_variant", ["overlap", "reverse"])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_peer_pcg_three_steps_owned_and_ghost_rows(ctx, P, map_variant, variant):
    """Three consecutive steps: every local row, owned and ghost, equals the
    oracle's third step -- ghost u, v come from the x (dv) rows the owners
    stored into the ghosts inside the kernel, and step 2 onwards maps the
    ghost tets with them.  The epoch counters and mailboxes carry over from
    launch to launch."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, iters, steps = 1e-2, 50, 3
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    u, v = case.u[order], case.vel[order]
    for _ in range(steps):
        ref = oracle.implicit_step(m, "nh", u, v, case.mu[tet_src], case.lam[tet_src], case.free[order], h,
                                   iters=iters)
        u, v = ref["u"], ref["v"]
    ranks = _ranks(ctx, case, P, f"pp3{P}{map_variant}{variant}", map_variant)
    peer = dist.PeerPCG(ranks, variant=variant)
    # reverse variant: the partial f / K rows of ghost tails go to their
    # owners as peer-memory REDs (PeerHalo ADD) -- no transport anywhere
    prev = (dist.PeerHalo(ranks, "rf"), dist.PeerHalo(ranks, "rK")) if map_variant == "reverse" else None
    u_in, v_in = np.empty_like(u), np.empty_like(v)
    u_in[order], v_in[order] = u, v
    for _ in range(steps):
        dist.implicit_step(ranks, None, "nh", h=h, iters=iters, variant="peer", peer=peer, peer_rev=prev)
    nghost = 0
    for R in ranks:
        ids, gu = R.local_values(R.fem.u)
        _, gv = R.local_values(R.fem.vel)
        ghost = ~R.owned_stored
        nghost += int(ghost.sum())
        assert rel_l2(gu, u_in[ids]) <= 1e-8
        assert rel_l2(gv, v_in[ids]) <= 1e-8
        assert rel_l2(gu[ghost], u_in[ids[ghost]]) <= 1e-8
        assert rel_l2(gv[ghost], v_in[ids[ghost]]) <= 1e-8
    assert nghost > 0


@pytest.mark.parametrize("variant", ["single", "saad"])
def test_peer_pcg_is_deterministic_and_split_launches_agree(ctx, variant):
    """Bitwise run-to-run deterministic (rank-ordered sums of deterministic
    per-CTA partials), and 50 iterations as 20 + 30 (two launches: the
    recurrences and the parity of the u buffers resume from the device
    scalars) equal one launch of 50 to round-off."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    ranks = _ranks(ctx, case, 3, f"ppdet{variant}")
    peer = dist.PeerPCG(ranks, variant=variant)
    outs = []
    for split in ([50], [50], [20, 30]):
        for R in ranks:
            R.map_assemble("nh", 1e-2, 0.0, 0.0, (0.0, -9.81, 0.0))
            R.cg_init(single=variant == "single")
        for k in split:
            peer.step(k)
        outs.append(np.concatenate([R.fem.dv.read().ravel() for R in ranks]))
    assert np.array_equal(outs[0], outs[1])
    assert rel_l2(outs[2], outs[0]) <= 1e-12


@pytest.mark.parametrize("variant", ["single", "saad"])
def test_peer_pcg_honours_the_tolerance(ctx, variant):
    """ebb_cg.tol > 0: every rank stops at the oracle's stop iteration (read
    off the single-domain r.z history), the same iterate."""
    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    h, P, tol = 1e-2, 3, 1e-3
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], h, iters=1)
    _, hist, _ = oracle.pcg(m.row_ptr, m.head, ref["A"], ref["b"], case.free[order], 300)
    thr = tol * tol * hist[0]
    k = next(k for k in range(1, 301) if hist[k] <= thr)
    assert abs(hist[k] - thr) > 1e-6 * thr and abs(hist[k - 1] - thr) > 1e-6 * thr
    x_ref, _, _ = oracle.pcg(m.row_ptr, m.head, ref["A"], ref["b"], case.free[order], k)
    ranks = _ranks(ctx, case, P, f"pptol{variant}")
    for R in ranks:
        R.fem.cg.tol = tol
    peer = dist.PeerPCG(ranks, variant=variant)
    for R in ranks:
        R.map_assemble("nh", h, 0.0, 0.0, (0.0, -9.81, 0.0))
        R.cg_init(single=variant == "single")
    peer.step(k + 40)
    peer.step(10)                                  # a no-op after the stop
    dv = _gather(ranks, "dv", m.nv)
    for R in ranks:
        assert R.fem.cg_iterations() == (k, True)
    assert rel_l2(dv[order], x_ref) <= 1e-8


@pytest.mark.parametrize("variant", ["single", "saad"])
def test_peer_pcg_fp32_derived_tolerance(ctx, variant):
    """fp32 on 2 ranks against the oracle's fp64 step, at the perturbation
    bound of test_gpu_edge_cases.test_pcg_fp32_50_iterations_derived_tolerance
    (kappa of the Jacobi-scaled free system, north_star fp32 bars)."""
    from test_gpu_edge_cases import _jacobi_condition

    from paper_1506_07577_b200 import dist
    case = Case(n=4, model="nh")
    for a in ("u", "mu", "lam", "vel"):
        setattr(case, a, getattr(case, a).astype(np.float32).astype(np.float64))
    m, new_of_old, tet_src, order = oracle_renumbered(case)
    ref = oracle.implicit_step(m, "nh", case.u[order], case.vel[order], case.mu[tet_src], case.lam[tet_src],
                               case.free[order], 1e-2, iters=50)
    kappa = _jacobi_condition(m, ref["A"], case.free[order])
    tol = kappa * (1e-5 + 1e-5) + 40.0 * kappa * 2.0 ** -24
    assert tol < 1e-3
    ranks = _ranks(ctx, case, 2, f"pp32{variant}", dtype="f32")
    peer = dist.PeerPCG(ranks, variant=variant)
    dist.implicit_step(ranks, None, "nh", h=1e-2, iters=50, variant="peer", peer=peer)
    assert rel_l2(_gather(ranks, "dv", m.nv)[order], ref["dv"]) <= tol


def test_peer_send_csr_matches_the_partition_lists(ctx):
    """ebb_peer_send_csr: per owned vertex, its (peer, remote row) entries in
    peer order -- equal to the CSR built here from the oracle's O4 lists, and
    every remote row names the same global vertex on the peer."""
    from paper_1506_07577_b200 import dist
    case = Case(n=5, model="nh")
    P = 4
    ranks = _ranks(ctx, case, P, "ppcsr")
    dist.PeerPCG(ranks)
    for R in ranks:
        off = R.peer_off.read().astype(np.int64).ravel()
        dst = R.peer_dst.read().astype(np.int64).reshape(-1, 2)
        assert off.size == R.n_owned + 1
        exp = {v: [] for v in range(R.n_owned)}
        for q in sorted(R.part_send):
            for k, v in enumerate(R.part_send[q]):
                exp[int(v)].append((q, int(ranks[q].part_recv[R.rank][k])))
        got_n = 0
        for v in range(R.n_owned):
            ent = [tuple(e) for e in dst[off[v]:off[v + 1]]]
            assert ent == exp[v]
            got_n += len(ent)
            for q, row in ent:
                assert ranks[q].verts_g[row] == R.verts_g[v]        # the same global vertex
        assert got_n == sum(len(r) for r in R.part_send.values())


def test_peer_bind_refuses_bad_arguments(ctx):
    import ctypes as C

    from paper_1506_07577_b200 import _abi as A
    from paper_1506_07577_b200 import dist
    from paper_1506_07577_b200.ebb import EbbError
    case = Case(n=4, model="nh")
    ranks = _ranks(ctx, case, 2, "ppbad")
    for R in ranks:
        R.peer_export(ipc=False)
    L, h = ctx.L, ctx.h
    g = C.c_int32()
    cgs = (A.CG * 2)(ranks[0].fem.cg, ranks[1].fem.cg)
    pcs = (A.PeerCG * 2)()
    for i, R in enumerate(ranks):
        off, dst = R.peer_send_csr(sorted(R.part_send), [ranks[q].part_recv[i] for q in sorted(R.part_send)],
                                   [ranks[q].fem.nv for q in sorted(R.part_send)])
        pcs[i].nranks, pcs[i].rank, pcs[i].n_owned = 2, i, R.n_owned
        pcs[i].send_off, pcs[i].send_dst, pcs[i].mbox = off.h, dst.h, R.mbox.h
    with pytest.raises(EbbError, match="EBB_E_ARG"):           # peer addresses missing
        ctx.check(L.ebb_cg_peer_bind(h, 2, cgs, pcs, C.byref(g)))
    pcs[1].rank = 0
    with pytest.raises(EbbError, match="EBB_E_ARG"):           # a rank bound twice / bad nranks
        ctx.check(L.ebb_cg_peer_bind(h, 2, cgs, pcs, C.byref(g)))
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        ctx.check(L.ebb_cg_peer_step(h, 99, 1, None))
    # out-of-range rows in the send lists
    R = ranks[0]
    q = sorted(R.part_send)[0]
    with pytest.raises(EbbError, match="EBB_E_RANGE"):
        R.peer_send_csr([q], [np.full(len(R.part_send[q]), 10 ** 6)], [ranks[q].fem.nv])
    with pytest.raises(EbbError, match="EBB_E_SIZE"):          # remote list of another length
        R.peer_send_csr([q], [np.zeros(len(R.part_send[q]) + 1, np.int64)], [ranks[q].fem.nv])
    # a halo group is not a PCG group and vice versa
    halo = dist.PeerHalo(ranks)
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        ctx.check(L.ebb_cg_peer_step(h, halo.group, 1, None))
    pcg = dist.PeerPCG(ranks)
    with pytest.raises(EbbError, match="EBB_E_ARG"):
        ctx.check(L.ebb_peer_halo_push(h, pcg.group, None))
    # a group whose field was freed refuses to launch
    peer = dist.PeerPCG(ranks)
    ranks[1].mbox.free()
    with pytest.raises(EbbError, match="EBB_E_STATE"):
        peer.step(1)


@pytest.mark.parametrize("variant", ["single", "saad"])
def test_peer_pcg_blob_mesh(ctx, variant):
    """The C3 blob (irregular boundary, ragged partitions, vertices of very
    different degree) over 3 emulated ranks: two consecutive steps equal the
    single-domain oracle on owned and ghost rows."""
    from synth import mesh as M
    from synth import state as S

    from paper_1506_07577_b200 import dist
    X, tets, n = M.blob(target_T=6_000)
    free = S.fixed_mask(X, n)
    u = S.twist_u(X, n, 6, free=free)
    mu, lam = S.materials(tets.shape[0], 2e5, 0.3, spread=0.1)
    vel = np.zeros_like(X)
    new_of_old, tet_src, tets_new = oracle.renumber(X, tets)
    order = np.argsort(new_of_old)
    m = oracle.Mesh(X[order], tets_new)
    uo, vo = u[order], vel[order]
    for _ in range(2):
        ref = oracle.implicit_step(m, "nh", uo, vo, mu[tet_src], lam[tet_src], free[order], 1e-2, iters=50)
        uo, vo = ref["u"], ref["v"]
    u_ref = np.empty_like(uo)
    u_ref[order] = uo
    ranks = []
    for r in range(3):
        part = dist.partition_rank(ctx, X, tets, 3, r, name=f"ppblob{variant}p{r}")
        ranks.append(dist.GpuRank(ctx, r, part, X, free, u, vel, mu, lam, name=f"ppblob{variant}r{r}", nranks=3))
    peer = dist.PeerPCG(ranks, variant=variant)
    for _ in range(2):
        dist.implicit_step(ranks, None, "nh", h=1e-2, iters=50, variant="peer", peer=peer)
    for R in ranks:
        ids, gu = R.local_values(R.fem.u)
        assert rel_l2(gu, u_ref[ids]) <= 1e-8


def test_peer_pcg_twenty_steps_track_the_single_domain_solve(ctx):
    """Long run: 20 consecutive distributed steps (3 emulated ranks, the
    fused peer PCG, auto body) stay on the single-domain GPU trajectory
    (TetFEM.implicit_step, the bench's single-GPU path) on every local row --
    ghost state that drifted a little each step would show up here."""
    from helpers import gpu_fem

    from paper_1506_07577_b200 import dist
    case = Case(n=6, model="nh", vel_amp=0.05)
    fem = gpu_fem(ctx, case, name="pp20ref")
    ranks = _ranks(ctx, case, 3, "pp20")
    peer = dist.PeerPCG(ranks)
    for _ in range(20):
        fem.implicit_step("nh", h=1e-2, iters=50)
        dist.implicit_step(ranks, None, "nh", h=1e-2, iters=50, variant="peer", peer=peer)
    u_ref = fem.to_input_order(fem.u.read())
    v_ref = fem.to_input_order(fem.vel.read())
    for R in ranks:
        ids, gu = R.local_values(R.fem.u)
        _, gv = R.local_values(R.fem.vel)
        assert rel_l2(gu, u_ref[ids]) <= 1e-8
        assert rel_l2(gv, v_ref[ids]) <= 1e-8
