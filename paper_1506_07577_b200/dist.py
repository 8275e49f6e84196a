"""Multi-GPU domain decomposition of the tet-FEM hot path.

Decomposition ("owner computes" with ghost tets):
  * owner maps follow O4 (``ebb_partition`` on the device, ``oracle.partition``
    in tests): tets in equal contiguous SFC ranges, every vertex owned by the
    rank of its lowest incident tet;
  * rank r holds every tet touching a vertex it owns (owned + ghost tets) and
    all their vertices (owned + ghost vertices).  Every edge row whose tail is
    owned is then complete locally, so the element map needs no reverse
    exchange (SURVEY §8(e) "alternative: overlapping decomposition");
  * the local problem -- local tets, local vertices (owned ascending, then
    ghosts), the tets' local keys and the halo lists of every peer -- is built
    on the device by ``ebb_partition_local`` (partition_rank below); each
    rank reads back only its own local-size arrays and frees the global mesh;
  * the PCG solves on owned rows only (mask = free AND owned).  Ghost copies
    of x, p, u, v stay consistent because they are updated with the same
    global alpha/beta from owner-consistent z, so per iteration the only
    exchanges are the z halo (owners -> ghosts) and two scalar sums (p.q,
    r.z).  Step order: map, assemble, cg_init, [sum rho/pq/rz, z halo],
    50 x (DIR, MATVEC, [sum p.q], UPDATE, [sum r.z, z halo]), state update.

The driver below is backend-agnostic: a *rank* object runs the local phases
(``GpuRank`` through the Ebb C ABI; the CPU test rank in tests/ through the
oracle) and a *transport* moves scalars and halo rows (``TorchTransport`` over
torch.distributed -- NCCL on B200s, gloo on CPU -- or ``LocalTransport`` for
several ranks driven from one process).
"""
from __future__ import annotations

import numpy as np

SLOT_RHO, SLOT_PQ, SLOT_RZ = 0, 1, 2
SLOT_RZ0, SLOT_DSUM, SLOT_GSUM = 7, 10, 11      # (solver.cu scalar slots)
CG_SR_PHASE = 3                                  # EBB_CG_SR_PHASE


# ----------------------------------------------------------------------------- transports
class TorchTransport:
    """torch.distributed collectives (NCCL on GPUs, gloo on CPU); one local rank."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def allreduce(self, ranks, slots):
        (R,) = ranks
        t = R.scal_tensor()
        lo, hi = slots
        v = t[lo:hi].clone()
        self.dist.all_reduce(v, group=self.group)
        t[lo:hi] = v

    def exchange(self, ranks):
        (R,) = ranks
        ops = []
        recvs = {}
        for peer in R.send_peers():
            ops.append(self.dist.P2POp(self.dist.isend, R.pack(peer), peer, group=self.group))
        for peer in R.recv_peers():
            rb = R.recv_buffer(peer)
            ops.append(self.dist.P2POp(self.dist.irecv, rb, peer, group=self.group))
            recvs[peer] = rb
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        for peer, rb in recvs.items():
            R.unpack(peer, rb)


class NcclTransport:
    """NCCL inside the library (ebb_comm_*): scalar allreduce and the grouped
    halo send/recv are stream-ordered library calls on the rank's stream; no
    torch collective on the iteration path.  The NCCL unique id is created by
    rank 0 and shared through torch.distributed (only at construction)."""

    def __init__(self, ctx, rank, size, stream=None):
        import ctypes as C
        self.C = C
        self.ctx, self.rank, self.size, self.stream = ctx, rank, size, stream
        uid = C.create_string_buffer(128)
        if rank == 0:
            ctx.check(ctx.L.ebb_comm_unique_id(uid))
        if size > 1:
            import torch
            import torch.distributed as dist
            t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
            dev = torch.device("cuda", ctx.device) if dist.get_backend() == "nccl" else torch.device("cpu")
            t = t.to(dev)
            dist.broadcast(t, 0)
            uid = C.create_string_buffer(bytes(t.cpu().tolist()), 128)
        ctx.check(ctx.L.ebb_comm_init(ctx.h, int(size), int(rank), uid))

    def _s(self):
        from .ebb import _stream
        return _stream(self.stream)

    def allreduce(self, ranks, slots):
        (R,) = ranks
        t = R.scal_tensor()
        lo, hi = slots
        self.ctx.check(self.ctx.L.ebb_comm_allreduce_sum(self.ctx.h, t.data_ptr() + 8 * lo, hi - lo, self._s()))

    def exchange(self, ranks):
        (R,) = ranks
        C = self.C
        peers = R.peers()
        if not peers:
            return
        n = len(peers)
        sp, rp = set(R.send_peers()), set(R.recv_peers())
        sb = [R.pack(p) if p in sp else None for p in peers]        # a direction may be empty
        rb = [R.recv_buffer(p) if p in rp else None for p in peers]
        nb = lambda b: 0 if b is None else b.numel() * b.element_size()
        ptr = lambda b: 0 if b is None else b.data_ptr()
        P = (C.c_int32 * n)(*peers)
        SP = (C.c_void_p * n)(*[ptr(b) for b in sb])
        SN = (C.c_uint64 * n)(*[nb(b) for b in sb])
        RP = (C.c_void_p * n)(*[ptr(b) for b in rb])
        RN = (C.c_uint64 * n)(*[nb(b) for b in rb])
        self.ctx.check(self.ctx.L.ebb_comm_halo(self.ctx.h, n, P, SP, SN, RP, RN, self._s()))
        for p, b in zip(peers, rb):
            if b is not None:
                R.unpack(p, b)


class LocalTransport:
    """Several ranks driven from one process (virtual shards on one device)."""

    def allreduce(self, ranks, slots):
        lo, hi = slots
        tot = None
        for R in ranks:
            v = R.scal_tensor()[lo:hi]
            tot = v.clone() if tot is None else tot + v
        for R in ranks:
            R.scal_tensor()[lo:hi] = tot

    def exchange(self, ranks):
        packed = {(R.rank, peer): R.pack(peer) for R in ranks for peer in R.send_peers()}
        for R in ranks:
            for peer in R.recv_peers():
                R.unpack(peer, packed[(peer, R.rank)])


# ----------------------------------------------------------------------------- driver
def _reverse_add(ranks, transport, peer_rev):
    """The partial f and K rows of ghost tails into their owners: the peer
    RED pushes (``peer_rev`` = (PeerHalo "rf", PeerHalo "rK")) or two
    transport exchanges."""
    if peer_rev is not None:
        for hp in peer_rev:
            hp.push()
        return
    for which in ("rf", "rK"):
        for R in ranks:
            R.set_halo(which)
        transport.exchange(ranks)


def _map_assemble(ranks, transport, model, h, alpha, beta, g, peer_rev=None):
    """The element map on every rank; with the reverse-add variant the partial
    f and K rows of ghost tails are added into their owners before the
    assembly reads them."""
    for R in ranks:
        R.map_forces(model)
    if getattr(ranks[0], "map_variant", "overlap") == "reverse":
        _reverse_add(ranks, transport, peer_rev)
    for R in ranks:
        R.assemble(h, alpha, beta, g)


def map_step(ranks, transport, model="stvk", halo=None, peer_rev=None):
    """The distributed element map alone (BASELINE configs[2]: the force +
    stiffness map with halo exchange): the owners' displacements go to their
    ghost copies (the position halo, owners -> ghosts), then every rank maps
    its tets -- with the reverse-add variant the partial f / K rows of ghost
    tails are added into their owners afterwards.  halo: a ``PeerHalo`` of
    the displacements -- the position halo as one peer-memory push kernel
    instead of the transport's pack / send / unpack."""
    if halo is not None:
        halo.push()
    else:
        for R in ranks:
            R.set_halo("disp")
        transport.exchange(ranks)
    for R in ranks:
        R.map_forces(model)
    if getattr(ranks[0], "map_variant", "overlap") == "reverse":
        _reverse_add(ranks, transport, peer_rev)


def implicit_step(ranks, transport, model="nh", h=1e-2, iters=50, alpha=0.0, beta=0.0, g=(0.0, -9.81, 0.0),
                  variant="saad", peer=None, peer_rev=None):
    """One distributed implicit step (O9 + O10) over `ranks` (the local ones).

    variant="saad": per iteration DIR, MATVEC, [sum p.q], UPDATE, [sum r.z,
    z halo] -- two scalar allreduces.  Ghost x is formed from the exchanged z
    with the global alpha/beta, so it stays equal to its owner's.

    variant="single": the single-reduction (Chronopoulos-Gear) recurrences in
    phase mode, per iteration ONE phase, ONE fused allreduce of (w.z, r.z) and
    the halo of the gathered operand u; iters iterations =
    iters + 1 phases (w_0 = A z_0 first).  Phase k writes u into buffer k % 2
    (solver.cu k_cg1_persistent: the parity flips as each phase finishes the
    previous recurrences), so only that buffer is exchanged.  Ghost rows are
    masked, so the kernel leaves ghost x at 0: x (= dv) is exchanged from the
    owners once, before the state update, so ghost u and v stay consistent
    for the next step's map on ghost tets.

    variant="peer": the same recurrences in ONE fused kernel for all
    iterations (ebb_cg_peer_step, bound by ``PeerPCG``): the owners store u,
    x (and z_0) into their peers' ghost rows and the two scalars go through
    peer mailboxes inside the kernel -- no host loop, no NCCL call, no
    transport (``transport`` is used only by the reverse-add map)."""
    _map_assemble(ranks, transport, model, h, alpha, beta, g, peer_rev)
    if variant == "peer":
        # the fused multi-GPU PCG: one kernel for every iteration (and the
        # z_0 / u / x halos and the scalar sums inside it); `peer` is the
        # PeerPCG binding of these ranks
        if peer is None:
            raise ValueError("variant='peer' needs the PeerPCG binding of the ranks")
        for R in ranks:
            R.cg_init(single=peer.variant == "single")
        peer.step(iters)
        for R in ranks:
            R.finish(h)
        return
    if variant == "single":
        for R in ranks:
            R.cg_init(single=True)
        transport.allreduce(ranks, (SLOT_RHO, SLOT_RZ + 1))
        transport.allreduce(ranks, (SLOT_RZ0, SLOT_RZ0 + 1))
        for R in ranks:
            R.set_halo("z")
        transport.exchange(ranks)
        nphase = iters + 1
        for k in range(nphase):
            for R in ranks:
                R.cg_phase(CG_SR_PHASE)
            transport.allreduce(ranks, (SLOT_DSUM, SLOT_GSUM + 1))
            if k + 1 < nphase:                 # the last phase's u is never gathered
                for R in ranks:
                    R.set_halo("u" if k % 2 == 0 else "u2")
                transport.exchange(ranks)
        for R in ranks:
            R.set_halo("x")
        transport.exchange(ranks)
        for R in ranks:
            R.finish(h)
        return
    for R in ranks:
        R.cg_init()
    transport.allreduce(ranks, (SLOT_RHO, SLOT_RZ + 1))
    for R in ranks:
        R.set_halo("z")
    transport.exchange(ranks)
    for _ in range(iters):
        for R in ranks:
            R.cg_phase(0)
        for R in ranks:
            R.cg_phase(1)
        transport.allreduce(ranks, (SLOT_PQ, SLOT_PQ + 1))
        for R in ranks:
            R.cg_phase(2)
        transport.allreduce(ranks, (SLOT_RZ, SLOT_RZ + 1))
        transport.exchange(ranks)
    for R in ranks:
        R.finish(h)


# ----------------------------------------------------------------------------- GPU setup
def partition_rank(ctx, X, tets, nranks, rank, name="part", mode="overlap", debug=False):
    """This rank's local problem, built on the device: upload the global mesh
    (positions and tets.v only -- no edge relation), orient (O1), renumber
    (a2: Morton vertices, tets by vertex tuple), the O4 owner maps
    (``ebb_partition``) and the local extraction (``ebb_partition_local``);
    read back the local-size arrays, free every global relation.

    Returns dict(vert_src, tet_src: the local vertices / tets as rows of the
    INPUT X / tets; vert_gid: the local vertices' global (renumbered, O3)
    ids; tets: the local tets in local vertex ids; n_owned: local
    vertices [0, n_owned) are owned; send / recv: {peer: local vertex rows};
    owner_v: the global owner map in stored order (tests); vert_order /
    tet_order: stored -> input rows of the global mesh (tests))."""
    import ctypes as C

    from . import _abi as A
    X = np.ascontiguousarray(X, dtype=np.float64)
    tets = np.ascontiguousarray(tets, dtype=np.int64)
    nv, nt = X.shape[0], tets.shape[0]
    L, h = ctx.L, ctx.h
    V = ctx.relation(f"{name}.gverts", nv)
    T = ctx.relation(f"{name}.gtets", nt)
    pos = V.field("pos", "f64", (3, 1), init=X)
    vid = V.field("orig_id", "u32", init=np.arange(nv, dtype=np.uint32))
    tid = T.field("orig_id", "u32", init=np.arange(nt, dtype=np.uint32))
    v = T.key_field("v", V, (4, 1), tets)
    sw = C.c_uint64()
    ctx.check(L.ebb_tetmesh_orient(h, v.h, pos.h, C.byref(sw)))
    ctx.check(L.ebb_renumber_morton(h, V.h, pos.h))
    ctx.check(L.ebb_sort_by_key_tuple(h, T.h, v.h))
    ot = T.field("owner_t", "i32")
    ov = V.field("owner_v", "i32")
    ctx.check(L.ebb_partition(h, v.h, int(nranks), ot.h, ov.h))
    info = A.PartitionInfo()
    sp = (C.c_uint64 * (nranks + 1))()
    rp = (C.c_uint64 * (nranks + 1))()
    ctx.check(L.ebb_partition_local(h, v.h, ot.h, ov.h, int(nranks), int(rank),
                                    A.PART_OVERLAP if mode == "overlap" else A.PART_OWN,
                                    f"{name}.r{rank}".encode(), C.byref(info), sp, rp))
    from .ebb import Field, Relation
    LT = Relation(ctx, info.ltets, f"{name}.r{rank}.ltets", info.n_ltets)
    LV = Relation(ctx, info.lverts, f"{name}.r{rank}.lverts", info.n_lverts)
    # input rows of the local vertices / tets: gather the global orig ids on the device
    vsrc = LV.field("src", "u32")
    tsrc = LT.field("src", "u32")
    ctx.check(L.ebb_rows_gather(h, vid.h, info.vert_gid, vsrc.h, None))
    ctx.check(L.ebb_rows_gather(h, tid.h, info.tet_gid, tsrc.h, None))
    out = dict(vert_src=vsrc.read().astype(np.int64), tet_src=tsrc.read().astype(np.int64),
               vert_gid=Field(ctx, info.vert_gid, LV, "gid", "u32", (1, 1), A.AOS).read().astype(np.int64),
               tets=Field(ctx, info.v, LT, "v", "key", (4, 1), A.AOS).read().astype(np.int64),
               n_owned=int(info.n_owned), send={}, recv={})
    for kind, rel, rows, ptr in (("send", info.send, info.send_rows, sp), ("recv", info.recv, info.recv_rows, rp)):
        if rel == A.NONE:
            continue
        R = Relation(ctx, rel, f"{name}.{kind}", int(ptr[nranks]))
        allrows = Field(ctx, rows, R, "rows", "u32", (1, 1), A.AOS).read().astype(np.int64)
        out[kind] = {q: allrows[ptr[q]:ptr[q + 1]] for q in range(nranks) if ptr[q + 1] > ptr[q]}
        R.free()
    if debug:
        out["owner_v"] = ov.read()
        out["vert_order"] = vid.read().astype(np.int64)
        out["tet_order"] = tid.read().astype(np.int64)
    LT.free()
    LV.free()
    T.free()
    V.free()
    return out


# ----------------------------------------------------------------------------- GPU rank
class GpuRank:
    """One rank's local problem on its GPU through the Ebb C ABI.

    part = partition_rank(...); X, free, u, vel (vertex rows) and mu, lam (tet
    rows) in the INPUT order of the global mesh.  The local mesh keeps the
    partition's order (owned vertices in global SFC order, then the ghosts;
    tets in global SFC order): no second renumbering, so the halo lists are
    local rows as they are.

    map_variant="overlap": every local tet is mapped (ghost tets recomputed,
    every owned row complete locally).  map_variant="reverse" (SURVEY §8(e) /
    north_star: "halo exchange of vertex positions and of the partial force
    sums"): each tet is mapped by ONE rank (the owner of its lowest-id
    vertex, ebb_partition_reverse); the partial f and K rows whose tail the
    rank does not own are added into their owners' rows (ebb_rows_scatter_add)
    before the assembly."""

    def __init__(self, ctx, rank, part, X, free, u, vel, mu, lam, rho=1e3, dtype="f64", stream=None, name=None,
                 map_variant="overlap", nranks=None):
        import torch

        from . import _abi as A
        from .tetfem import TetFEM
        vs, ts = part["vert_src"], part["tet_src"]
        n_owned = part["n_owned"]
        self.rank, self.ctx, self.stream, self.A = rank, ctx, stream, A
        self.dtype = dtype
        self.tdt = torch.float64 if dtype == "f64" else torch.float32
        self.verts_g = vs                              # input row of every local vertex
        self.vert_gid = part.get("vert_gid")           # global (renumbered) id of every local vertex
        owned = np.arange(vs.size) < n_owned
        mask = (np.asarray(free)[vs].astype(bool) & owned).astype(np.uint8)
        self.fem = TetFEM(ctx, np.asarray(X)[vs], part["tets"], dtype=dtype, mu=np.asarray(mu)[ts],
                          lam=np.asarray(lam)[ts], rho=rho, free=mask, u=np.asarray(u)[vs],
                          vel=np.asarray(vel)[vs], renumber=False, name=name or f"r{rank}")
        self.owned_stored = owned
        # allocates every CG work field (the single-reduction set includes u, u2)
        self.fem.cg_init(stream, variant=A.CG_SINGLE_REDUCTION)
        self.z_field = self._field(self.fem.cg.z, 4)
        # halo fields: padded CG vectors (4 components) and dv (x of the PCG, 3)
        self.halo_fields = {"z": self.z_field, "u": self._field(self.fem.cg.u, 4),
                            "u2": self._field(self.fem.cg.u2, 4), "x": self.fem.dv, "disp": self.fem.u}
        self.scal = self._field(self.fem.cg.scal, 1, count=12, dt="f64").tensor()
        self._lists = {}
        self.n_owned = int(n_owned)
        self.part_send, self.part_recv = part["send"], part["recv"]
        self._make_lists("fwd", self.fem.verts.name + ".halo", part["send"], part["recv"], (3, 4))
        self.map_variant = map_variant
        if map_variant == "reverse":
            self._setup_reverse(part, nranks if nranks is not None else 1 + max([rank, *part["send"],
                                                                                  *part["recv"]]))
        elif map_variant != "overlap":
            raise ValueError(map_variant)
        self.set_halo("z")
        torch.cuda.synchronize()

    def _make_lists(self, tag, prefix, send, recv, ncs):
        """Row lists + staging buffers (one per component count) per peer: the
        buffers are library fields on the list relation, seen by the
        transports as zero-copy torch views."""
        L = {"send": {}, "recv": {}}
        for kind, lists in (("send", send), ("recv", recv)):
            for peer, rows in lists.items():
                rel = self.ctx.relation(f"{prefix}.{tag}.{kind}{peer}", len(rows))
                rf = rel.field("rows", "u32", init=np.asarray(rows).astype(np.uint32))
                bufs = {}
                for nc in ncs:
                    bf = rel.field(f"buf{nc}", self.dtype, (nc, 1))
                    bufs[nc] = (bf, bf.tensor().view(len(rows), nc))
                L[kind][peer] = (rf, bufs)
        L["peers"] = sorted(set(L["send"]) | set(L["recv"]))
        self._lists[tag] = L

    def _setup_reverse(self, part, nranks):
        """The own-tet subset (tets this rank maps) sharing the local vertex and
        edge relations, and the reverse-add lists of f and K rows."""
        import ctypes as C

        from . import _abi as A
        ctx, fem = self.ctx, self.fem
        owner = np.full(fem.nv, self.rank, dtype=np.int32)
        for q, rows in part["recv"].items():
            owner[rows] = q
        # the key every rank shares for "the tet's lowest vertex" and the list
        # order: the INPUT row ids (scrambled w.r.t. the SFC order, so the
        # computing ranks stay balanced; with the renumbered ids the lowest
        # vertex's owner is biased towards the lower ranks -- measured: the
        # last rank computes no foreign rows and the map's slowest rank is
        # 3-10 % slower, profiles/r02_dist_variants_renumbered_key.jsonl)
        gid = fem.verts.field("gid", "u32", init=np.asarray(self.verts_g).astype(np.uint32))
        own_f = fem.verts.field("owner", "i32", init=owner)
        info = A.ReverseInfo()
        ptr = (C.c_uint64 * (4 * (nranks + 1)))()
        ctx.check(ctx.L.ebb_partition_reverse(ctx.h, fem.v.h, fem.e.h, gid.h, own_f.h, int(nranks), int(self.rank),
                                              f"{fem.verts.name}.rev".encode(), C.byref(info), ptr))
        from .ebb import Field, Relation
        own = Field(ctx, info.own, fem.tets, "own", "u8", (1, 1), A.AOS).read().astype(bool)
        lists = []
        for k, (rel, rows) in enumerate(((info.fsend, info.fsend_rows), (info.frecv, info.frecv_rows),
                                          (info.ksend, info.ksend_rows), (info.krecv, info.krecv_rows))):
            p0 = k * (nranks + 1)
            d = {}
            if rel != A.NONE:
                R_ = Relation(ctx, rel, "rev", int(ptr[p0 + nranks]))
                allr = Field(ctx, rows, R_, "rows", "u32", (1, 1), A.AOS).read().astype(np.int64)
                d = {q: allr[ptr[p0 + q]:ptr[p0 + q + 1]] for q in range(nranks) if ptr[p0 + q + 1] > ptr[p0 + q]}
                R_.free()
            lists.append(d)
        self._make_lists("rf", fem.verts.name + ".rev", lists[0], lists[1], (3,))
        self._make_lists("rK", fem.verts.name + ".rev", lists[2], lists[3], (9,))
        self.rev_lists = {"rf": (lists[0], lists[1]), "rK": (lists[2], lists[3])}   # (send, recv) rows per peer
        # the own-tet subset: its own relation with keys into the local verts / edges
        sel = np.nonzero(own)[0]
        self.n_map_tets = int(sel.size)
        T2 = ctx.relation(f"{fem.tets.name}.own", max(int(sel.size), 1))
        self.map_fields = dict(
            v=T2.key_field("v", fem.verts, (4, 1), fem.v.read()[sel]),
            e=T2.key_field("e", fem.edges, (4, 4), fem.e.read().reshape(-1, 16)[sel]),
            Dminv=T2.field("Dminv", self.dtype, (3, 3), "soa", init=fem.Dminv.read().reshape(-1, 9)[sel]),
            W=T2.field("W", self.dtype, init=fem.W.read()[sel]),
            mu=T2.field("mu", self.dtype, init=fem.mu.read()[sel]),
            lam=T2.field("lam", self.dtype, init=fem.lam.read()[sel]))
        self.rev_bytes = {tag: sum(int(b[1][nc][1].numel()) * (8 if self.dtype == "f64" else 4)
                                   for b in self._lists[tag]["send"].values() for nc in b[1])
                          for tag in ("rf", "rK")}

    def _field(self, h, rows, count=None, dt=None):
        from .ebb import Field
        f = Field(self.ctx, h, self.fem.verts if count is None else None, "cgwork", dt or self.fem.dtype,
                  (rows, 1), self.A.AOS)
        if count is not None:
            f.count = count
        return f

    # -- phases
    def map_forces(self, model):
        if self.map_variant == "overlap":
            self.fem.map_forces(model, True, False, stream=self.stream)
            return
        import ctypes as C

        from . import _abi as A
        from .ebb import _stream
        from .tetfem import MODELS
        F = self.map_fields
        d = A.TetMapDesc()
        d.model, d.scatter, d.zero_outputs = MODELS[model], A.SCATTER_AUTO, 1
        d.v, d.e, d.u = F["v"].h, F["e"].h, self.fem.u.h
        d.Dminv, d.W, d.mu, d.lam = F["Dminv"].h, F["W"].h, F["mu"].h, F["lam"].h
        d.f, d.K, d.energy = self.fem.f.h, self.fem.K.h, A.NONE
        self.ctx.check(self.ctx.L.ebb_map_tet_forces(self.ctx.h, C.byref(d), _stream(self.stream)))

    def assemble(self, h, alpha, beta, g):
        self.fem.assemble(h, alpha, beta, g, stream=self.stream)

    def map_assemble(self, model, h, alpha, beta, g):
        self.map_forces(model)
        self.assemble(h, alpha, beta, g)

    def cg_init(self, single=False):
        from . import _abi as A
        self.fem.cg_init(self.stream, variant=A.CG_SINGLE_REDUCTION if single else A.CG_SAAD)

    def set_halo(self, which):
        """What the next exchange moves: a vertex field owners -> ghosts (z, u,
        u2, x), or the reverse add of partial rows ghost tails -> owners (rf:
        forces, rK: stiffness rows)."""
        if which in ("rf", "rK"):
            self._cur = self._lists[which]
            self.halo_field = self.fem.f if which == "rf" else self.fem.K
            self._add = True
        else:
            self._cur = self._lists["fwd"]
            self.halo_field = self.halo_fields[which]
            self._add = False

    def cg_phase(self, k):
        import ctypes as C

        from .ebb import _stream
        self.ctx.check(self.ctx.L.ebb_cg_phase(self.ctx.h, C.byref(self.fem.cg), int(k), _stream(self.stream)))

    def finish(self, h):
        from .ebb import _stream
        self.ctx.check(self.ctx.L.ebb_implicit_update(self.ctx.h, self.fem.dv.h, float(h), self.fem.u.h,
                                                      self.fem.vel.h, _stream(self.stream)))

    # -- fused PCG over peer memory (PeerPCG)
    def _list_rows(self, lists):
        """(send, recv) rows per peer and the relation rows of a list set:
        "fwd" (vertex halo), "rf" / "rK" (reverse add of forces / K rows)."""
        if lists == "fwd":
            return self.part_send, self.part_recv, int(self.fem.nv)
        send, recv = self.rev_lists[lists]
        return send, recv, int(self.fem.nv if lists == "rf" else self.fem.ne)

    def peer_export(self, ipc, extra=None, lists="fwd"):
        """What peers need of this rank: its recv rows per peer (numpy), its
        local vertex count, send-list lengths, and its ghost-row targets
        (cg.u, cg.u2, cg.x = dv, cg.z, the mailbox) as device addresses
        (ranks on one device) or 64-byte IPC handles (one process per GPU)."""
        import ctypes as C

        from . import _abi as A
        if not hasattr(self, "mbox"):
            rel = self.ctx.relation(f"{self.fem.verts.name}.mbox", A.PEER_MBOX_WORDS)
            self.mbox = rel.field("mbox", "f64", init=np.zeros(A.PEER_MBOX_WORDS))
        cg = self.fem.cg
        handles = {"u": cg.u, "u2": cg.u2, "x": cg.x, "z": cg.z, "mbox": self.mbox.h}
        handles.update(extra or {})
        buf = {}
        for name, fh in handles.items():
            if ipc:
                hb = C.create_string_buffer(64)
                self.ctx.check(self.ctx.L.ebb_ipc_handle(self.ctx.h, int(fh), hb))
                buf[name] = hb.raw
            else:
                v = A.View()
                self.ctx.check(self.ctx.L.ebb_field_view(self.ctx.h, int(fh), C.byref(v)))
                buf[name] = int(v.data)
        send, recv, nrows = self._list_rows(lists)
        return dict(rank=self.rank, nv=nrows, send={q: int(len(r)) for q, r in send.items()},
                    recv={q: np.asarray(r, np.int64) for q, r in recv.items()}, buf=buf)

    def peer_send_csr(self, peers, remote, peer_nv, lists="fwd"):
        """ebb_peer_send_csr over this rank's send lists of a list set (fields
        of the halo lists) and the peers' rows of the same rows."""
        import ctypes as C

        from . import _abi as A
        n = len(peers)
        self._peer_calls = getattr(self, "_peer_calls", 0) + 1
        tag = f"{self.fem.verts.name}.peer{self._peer_calls}"
        self._remote_rels = []
        sf, rf = [], []
        for q, rows in zip(peers, remote):
            rel = self.ctx.relation(f"{tag}.remote{q}", max(len(rows), 1))
            self._remote_rels.append(rel)
            rf.append(rel.field("rows", "u32", init=np.asarray(rows, np.uint32)).h)
            sf.append(self._lists[lists]["send"][q][0].h)
        off, dst = C.c_uint32(), C.c_uint32()
        n_src = self.n_owned if lists == "fwd" else self._list_rows(lists)[2]
        self.ctx.check(self.ctx.L.ebb_peer_send_csr(
            self.ctx.h, n_src, n, (C.c_int32 * max(n, 1))(*peers), (A.u32 * max(n, 1))(*sf),
            (A.u32 * max(n, 1))(*rf), (C.c_uint64 * max(n, 1))(*peer_nv), tag.encode(),
            C.byref(off), C.byref(dst)))
        from .ebb import Field
        po = Field(self.ctx, off.value, None, "off", "u32", (1, 1), A.AOS)
        po.count = n_src + 1
        pd = Field(self.ctx, dst.value, None, "dst", "u32", (2, 1), A.AOS)
        pd.count = max(sum(len(r) for r in remote), 1)
        if not hasattr(self, "peer_csr"):
            self.peer_csr = {}
        self.peer_csr[lists] = (po, pd, n_src)
        if lists == "fwd":
            self.peer_off, self.peer_dst = po, pd
        return po, pd

    # -- transport hooks
    def scal_tensor(self):
        return self.scal

    def peers(self):
        return self._cur["peers"]

    def send_peers(self):
        return sorted(self._cur["send"])

    def recv_peers(self):
        return sorted(self._cur["recv"])

    def _nc(self):
        return self.halo_field.shape[0] * self.halo_field.shape[1]

    def pack(self, peer):
        from .ebb import _stream
        rf, bufs = self._cur["send"][peer]
        bf, buf = bufs[self._nc()]
        self.ctx.check(self.ctx.L.ebb_rows_gather(self.ctx.h, self.halo_field.h, rf.h, bf.h, _stream(self.stream)))
        return buf

    def recv_buffer(self, peer):
        return self._cur["recv"][peer][1][self._nc()][1]

    def unpack(self, peer, data):
        from .ebb import _stream
        rf, bufs = self._cur["recv"][peer]
        bf, buf = bufs[self._nc()]
        if data is not buf:
            buf.copy_(data)
        fn = self.ctx.L.ebb_rows_scatter_add if self._add else self.ctx.L.ebb_rows_scatter
        self.ctx.check(fn(self.ctx.h, self.halo_field.h, rf.h, bf.h, _stream(self.stream)))

    # -- results in the input numbering of the global mesh
    def owned_values(self, field):
        vals = field.read()
        return self.verts_g[self.owned_stored], vals[self.owned_stored]

    def local_values(self, field):
        """Every local row (owned and ghost) with its input vertex id."""
        return self.verts_g, field.read()


# ----------------------------------------------------------------------------- fused PCG over peer memory
PEER_BUFFERS = ("u", "u2", "x", "z", "mbox")


def peer_tables(infos, local_ranks, nranks, names=PEER_BUFFERS):
    """What each local rank needs of its peers for ebb_cg_peer_bind, from the
    peers' exported infos (``GpuRank.peer_export``): per local rank r, the
    sorted send peers q with r's remote rows on q (q's recv rows from r: the
    same vertices in the same ascending-gid order, ebb_partition_local), q's
    local vertex count, and q's buffer entries (addresses or IPC handles).
    Pure host bookkeeping (no arithmetic of the method); checked on CPU."""
    out = {}
    for r in local_ranks:
        me = infos[r]
        peers = sorted(me["send"])
        remote, peer_nv = [], []
        for q in peers:
            rows = np.asarray(infos[q]["recv"].get(r, np.zeros(0, np.int64)))
            if rows.size != me["send"][q]:
                raise ValueError(f"rank {r} sends {me['send'][q]} rows to {q}, which expects {rows.size}")
            remote.append(rows)
            peer_nv.append(int(infos[q]["nv"]))
        bufs = {name: [infos[q]["buf"][name] if q != r else None for q in range(nranks)] for name in names}
        out[r] = dict(peers=peers, remote=remote, peer_nv=peer_nv, bufs=bufs)
    return out


class PeerPCG:
    """The fused multi-GPU PCG over peer memory (``ebb_cg_peer_bind`` /
    ``ebb_cg_peer_step``); variant "single" (single-reduction:
    one scalar exchange per iteration, u / x halo) or "saad" (two exchanges,
    z / x halo; the faster form once the vector records stream from HBM).

    ranks: the GpuRank objects of THIS process, all on one device.
    comm=None: every rank of the job is in ``ranks`` (ranks emulated on one
    device -- one cooperative launch runs all of them; the peers' buffers are
    addressed directly).  comm = a torch.distributed group: one rank per
    process and GPU; the peers' buffers are CUDA-IPC mapped (ebb_ipc_*), the
    infos travel once through ``all_gather_object``.  After binding, one
    ``step(iters)`` per implicit step replaces the per-phase launches,
    allreduces and halo exchanges of the "single" driver."""

    # the single-GPU AUTO crossover (solver.cu cg_variant):
    # single-reduction while a rank's vector records stay in L2
    AUTO_SINGLE_MAX_VERTS = 232000

    def __init__(self, ranks, comm=None, stream=None, variant="auto"):
        import ctypes as C

        from . import _abi as A
        if variant not in ("auto", "single", "saad"):
            raise ValueError(variant)
        self.ranks, self.ctx, self.stream = list(ranks), ranks[0].ctx, stream
        ctx = self.ctx
        ipc = comm is not None
        infos, nranks = _gather_infos(self.ranks, comm, lambda R: None)
        if variant == "auto":                 # the same choice on every rank: from the gathered sizes
            variant = "single" if max(d["nv"] for d in infos.values()) <= self.AUTO_SINGLE_MAX_VERTS else "saad"
        self.variant = variant
        for R in self.ranks:                  # the body the kernel runs (ebb_cg_peer_bind reads the variant)
            R.fem.cg.variant = A.CG_SINGLE_REDUCTION if variant == "single" else A.CG_SAAD
        tables = peer_tables(infos, [R.rank for R in self.ranks], nranks)
        self._opened = []
        self.peer_addr = {}                        # (local rank, peer, buffer) -> device address used
        cgs = (A.CG * len(self.ranks))()
        pcs = (A.PeerCG * len(self.ranks))()
        for i, R in enumerate(self.ranks):
            t = tables[R.rank]
            if "fwd" not in getattr(R, "peer_csr", {}):   # one send CSR per rank (a property of the partition)
                R.peer_send_csr(t["peers"], t["remote"], t["peer_nv"])
            off, dst = R.peer_off, R.peer_dst
            pc = pcs[i]
            pc.nranks, pc.rank, pc.n_owned = nranks, R.rank, R.n_owned
            pc.send_off, pc.send_dst, pc.mbox = off.h, dst.h, R.mbox.h
            for name, arr in (("u", pc.peer_u), ("u2", pc.peer_u2), ("x", pc.peer_x), ("z", pc.peer_z),
                              ("mbox", pc.peer_mbox)):
                for q, b in enumerate(t["bufs"][name]):
                    if b is None:
                        continue
                    if ipc:
                        addr = C.c_uint64()
                        ctx.check(ctx.L.ebb_ipc_open(ctx.h, bytes(b), C.byref(addr)))
                        self._opened.append(addr.value)
                        b = addr.value
                    arr[q] = int(b)
                    self.peer_addr[(R.rank, q, name)] = int(b)
            cgs[i] = R.fem.cg
        g = C.c_int32()
        ctx.check(ctx.L.ebb_cg_peer_bind(ctx.h, len(self.ranks), cgs, pcs, C.byref(g)))
        self.group = g.value
        if ipc:
            import torch.distributed as tdist
            tdist.barrier(group=comm)     # every rank mapped its peers before anyone steps

    def step(self, iters):
        from .ebb import _stream
        if self.group is None:
            raise RuntimeError("PeerPCG.step after close(): the peers' mappings are gone")
        self.ctx.check(self.ctx.L.ebb_cg_peer_step(self.ctx.h, self.group, int(iters), _stream(self.stream)))

    def close(self):
        """Unmap the peers' buffers (one process per GPU); the binding is
        unusable afterwards.  Every rank must have finished its last step
        first (a barrier), or a peer could still be storing into us."""
        for a in self._opened:
            self.ctx.check(self.ctx.L.ebb_ipc_close(self.ctx.h, a))
        self._opened = []
        self.group = None


def _gather_infos(ranks, comm, extra, lists="fwd"):
    """Every rank's peer infos (local: direct; one process per GPU: through
    all_gather_object) and the job's rank count."""
    ipc = comm is not None
    if ipc:
        import torch.distributed as tdist
        nranks = tdist.get_world_size(comm)
        (R0,) = ranks
        gathered = [None] * nranks
        tdist.all_gather_object(gathered, R0.peer_export(ipc=True, extra=extra(R0), lists=lists), group=comm)
        infos = {d["rank"]: d for d in gathered}
    else:
        nranks = len(ranks)
        infos = {R.rank: R.peer_export(ipc=False, extra=extra(R), lists=lists) for R in ranks}
    if sorted(infos) != list(range(nranks)):
        raise ValueError(f"peer ranks {sorted(infos)} are not 0..{nranks - 1}")
    return infos, nranks


class PeerHalo:
    """A halo of a field over peer memory (``ebb_peer_halo_bind`` /
    ``ebb_peer_halo_push``, SURVEY §8(e) "halo exchange of vertex positions
    and of the partial force sums").  which = "disp" (the displacements u,
    owners -> ghosts, copy), or "rf" / "rK" (map_variant="reverse": the
    partial force / stiffness rows of ghost tails added into their owners
    with red.global.add over peer memory).  One mailbox exchange before and
    one after the stores (shared with the ranks' PeerPCG epoch counter).
    comm as for ``PeerPCG``."""

    def __init__(self, ranks, which="disp", comm=None, stream=None):
        import ctypes as C

        from . import _abi as A
        self.ranks, self.ctx, self.stream = list(ranks), ranks[0].ctx, stream
        ctx = self.ctx
        ipc = comm is not None
        add = which in ("rf", "rK")
        lists = which if add else "fwd"
        field_of = (lambda R: R.fem.f) if which == "rf" else (lambda R: R.fem.K) if which == "rK" else \
            (lambda R: R.halo_fields[which])
        infos, nranks = _gather_infos(self.ranks, comm, lambda R: {"halo": field_of(R).h}, lists=lists)
        tables = peer_tables(infos, [R.rank for R in self.ranks], nranks, names=("halo", "mbox"))
        self._opened = []
        ds = (A.PeerHalo * len(self.ranks))()
        for i, R in enumerate(self.ranks):
            t = tables[R.rank]
            if lists not in getattr(R, "peer_csr", {}):
                R.peer_send_csr(t["peers"], t["remote"], t["peer_nv"], lists=lists)
            off, dst, n_src = R.peer_csr[lists]
            d = ds[i]
            d.nranks, d.rank, d.n_src = nranks, R.rank, n_src
            d.field, d.send_off, d.send_dst, d.mbox = field_of(R).h, off.h, dst.h, R.mbox.h
            d.mode = A.HALO_ADD if add else A.HALO_COPY
            for q in range(nranks):
                if q != R.rank:
                    d.peer_rows[q] = int(infos[q]["nv"])
            for name, arr in (("halo", d.peer_field), ("mbox", d.peer_mbox)):
                for q, b in enumerate(t["bufs"][name]):
                    if b is None:
                        continue
                    if ipc:
                        addr = C.c_uint64()
                        ctx.check(ctx.L.ebb_ipc_open(ctx.h, bytes(b), C.byref(addr)))
                        self._opened.append(addr.value)
                        b = addr.value
                    arr[q] = int(b)
        g = C.c_int32()
        ctx.check(ctx.L.ebb_peer_halo_bind(ctx.h, len(self.ranks), ds, C.byref(g)))
        self.group = g.value
        if ipc:
            import torch.distributed as tdist
            tdist.barrier(group=comm)

    def push(self):
        from .ebb import _stream
        if self.group is None:
            raise RuntimeError("PeerHalo.push after close()")
        self.ctx.check(self.ctx.L.ebb_peer_halo_push(self.ctx.h, self.group, _stream(self.stream)))

    def close(self):
        for a in self._opened:
            self.ctx.check(self.ctx.L.ebb_ipc_close(self.ctx.h, a))
        self._opened = []
        self.group = None
