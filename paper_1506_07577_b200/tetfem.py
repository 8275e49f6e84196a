"""Tetrahedral FEM domain + integrators on the Ebb C ABI.

``TetFEM`` builds the paper's FEM tetmesh domain -- relations ``verts``,
``tets``, ``edges`` (ordered pairs + a self-loop per vertex, grouped by tail),
key-fields ``tets.v[4]``, ``tets.e[4][4]``, ``edges.tail/head`` -- then runs
the hot path: the element force/stiffness map, the implicit (Vega-style
backward Euler + Jacobi-PCG) step, or the Fig. 2 explicit update.  Each method
is a short sequence of ``ebb_*`` calls; no arithmetic happens in Python.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from .ebb import Context, _stream

MODELS = {"stvk": A.STVK, "nh": A.NH}


class TetFEM:
    """Device-resident FEM state for one mesh on one GPU.

    Inputs are in the caller's vertex / tet order; with ``renumber=True`` the
    runtime reorders both relations for locality (Morton order of the rest
    positions, tets by sorted vertex tuple; licence P:674-677).  ``vert_order``
    and ``tet_order`` give the caller's index of every stored row.
    """

    def __init__(self, ctx: Context, X, tets, *, dtype="f64", mu=None, lam=None, rho=1e3, free=None,
                 u=None, vel=None, renumber=True, orient=True, mass="lumped", name="mesh"):
        self.ctx = ctx
        self.dtype = dtype
        X = np.ascontiguousarray(X, dtype=np.float64)
        tets = np.ascontiguousarray(tets, dtype=np.int64)
        self.nv, self.nt = X.shape[0], tets.shape[0]
        r = ctx.relation
        self.verts = r(f"{name}.verts", self.nv)
        self.tets = r(f"{name}.tets", self.nt)
        V, T = self.verts, self.tets
        self.pos = V.field("pos", "f64", (3, 1), init=X)
        self.vid = V.field("orig_id", "u32", (1, 1), init=np.arange(self.nv, dtype=np.uint32))
        self.u = V.field("u", dtype, (3, 1), init=u if u is not None else np.zeros((self.nv, 3)))
        self.vel = V.field("vel", dtype, (3, 1), init=vel if vel is not None else np.zeros((self.nv, 3)))
        self.free = V.field("free", "u8", (1, 1), init=free if free is not None else np.ones(self.nv, np.uint8))
        self.has_mask = free is not None
        self.tid = T.field("orig_id", "u32", (1, 1), init=np.arange(self.nt, dtype=np.uint32))
        mu = np.full(self.nt, 1.0) if mu is None else mu
        lam = np.full(self.nt, 1.0) if lam is None else lam
        self.mu = T.field("mu", dtype, (1, 1), init=mu)
        self.lam = T.field("lam", dtype, (1, 1), init=lam)
        self.v = T.key_field("v", V, (4, 1), tets)
        L, h = ctx.L, ctx.h
        if orient:
            sw = C.c_uint64()
            ctx.check(L.ebb_tetmesh_orient(h, self.v.h, self.pos.h, C.byref(sw)))
            self.swaps = sw.value
        if renumber:
            ctx.check(L.ebb_renumber_morton(h, V.h, self.pos.h))
            ctx.check(L.ebb_sort_by_key_tuple(h, T.h, self.v.h))
        out = A.TetmeshOut()
        ctx.check(L.ebb_tetmesh_build(h, self.v.h, f"{name}.edges".encode(), C.byref(out)))
        self.mesh = out
        ne = C.c_uint64()
        ctx.check(L.ebb_relation_size(h, out.edges, C.byref(ne)))
        self.ne = ne.value
        from .ebb import Field, Relation
        self.edges = Relation(ctx, out.edges, f"{name}.edges", self.ne)
        self.tail = Field(ctx, out.tail, self.edges, "tail", "key", (1, 1), A.AOS)
        self.head = Field(ctx, out.head, self.edges, "head", "key", (1, 1), A.AOS)
        self.e = Field(ctx, out.e, T, "e", "key", (4, 4), A.AOS)
        self.self_e = Field(ctx, out.self, V, "self", "key", (1, 1), A.AOS)
        self.index = Field(ctx, out.index, None, "__index", "u32", (1, 1), A.AOS)
        self.index.count = self.nv + 1
        # rest data (a3) in fp64, converted to the map dtype
        Dm64 = T.field("Dminv64", "f64", (3, 3), "soa")
        W64 = T.field("W64", "f64")
        m64 = V.field("mass64", "f64")
        ctx.check(L.ebb_tetmesh_rest(h, self.v.h, self.pos.h, float(rho), Dm64.h, W64.h, m64.h, None))
        if dtype == "f64":
            self.Dminv, self.W, self.mass = Dm64, W64, m64
        else:
            self.Dminv = T.field("Dminv", dtype, (3, 3), "soa")
            self.W = T.field("W", dtype)
            self.mass = V.field("mass", dtype)
            self.Dminv.convert_from(Dm64)
            self.W.convert_from(W64)
            self.mass.convert_from(m64)
        # mass="consistent": the Galerkin mass on the edge relation,
        # used by assemble() in place of the lumped vertex mass
        self.mass_kind = mass
        if mass == "consistent":
            me64 = self.edges.field("mass_e64", "f64")
            ctx.check(L.ebb_tetmesh_consistent_mass(h, self.e.h, W64.h, float(rho), me64.h, None))
            if dtype == "f64":
                self.mass_e = me64
            else:
                self.mass_e = self.edges.field("mass_e", dtype)
                self.mass_e.convert_from(me64)
        elif mass != "lumped":
            raise ValueError(f"mass must be 'lumped' or 'consistent', not {mass!r}")
        # per-step fields
        self.f = V.field("f", dtype, (3, 1))
        self.K = self.edges.field("K", dtype, (3, 3), "soa")
        self.b = V.field("b", dtype, (3, 1))
        self.dv = V.field("dv", dtype, (3, 1))
        self.energy = ctx.global_(f"{name}.energy", dtype)
        self.cg = None
        ctx.sync()

    # ---------------------------------------------------------------- orders
    def vert_order(self):
        return self.vid.read().astype(np.int64)

    def tet_order(self):
        return self.tid.read().astype(np.int64)

    def to_input_order(self, arr_stored):
        """Vertex field in stored order -> caller order."""
        out = np.empty_like(arr_stored)
        out[self.vert_order()] = arr_stored
        return out

    def from_input_order(self, arr_in):
        return np.ascontiguousarray(arr_in[self.vert_order()])

    # ---------------------------------------------------------------- hot path
    def plan_stats(self):
        """Statistics of the SEGMENTED map plan of this mesh (after a map)."""
        return self.ctx.map_plan_stats(self.v.h, self.e.h)

    def chunk_stats(self):
        """Statistics of the CHUNK map plan of this mesh (after a CHUNK map)."""
        return self.ctx.map_chunk_stats(self.v.h, self.e.h)

    def map_forces(self, model="nh", want_K=True, want_energy=True, scatter=A.SCATTER_AUTO, zero_outputs=True,
                   stream=None):
        d = A.TetMapDesc()
        d.model = MODELS[model]
        d.scatter = scatter
        d.zero_outputs = int(zero_outputs)
        d.v, d.e, d.u = self.v.h, self.e.h, self.u.h
        d.Dminv, d.W, d.mu, d.lam = self.Dminv.h, self.W.h, self.mu.h, self.lam.h
        d.f = self.f.h
        d.K = self.K.h if want_K else A.NONE
        d.energy = self.energy.h if want_energy else A.NONE
        self.ctx.check(self.ctx.L.ebb_map_tet_forces(self.ctx.h, C.byref(d), _stream(stream)))

    def _map_desc(self, model):
        d = A.TetMapDesc()
        d.model = MODELS[model]
        d.v, d.e, d.u = self.v.h, self.e.h, self.u.h
        d.Dminv, d.W, d.mu, d.lam = self.Dminv.h, self.W.h, self.mu.h, self.lam.h
        d.f, d.K, d.energy = self.f.h, A.NONE, A.NONE
        return d

    def ebe_state(self, model="nh", stream=None):
        """the compact per-tet stiffness state at the current u."""
        words = 15 if model == "nh" else 26
        key = f"ebe_state_{model}"
        if getattr(self, key, None) is None:
            setattr(self, key, self.tets.field(key, self.dtype, (words, 1), "soa"))
        st = getattr(self, key)
        self.ctx.check(self.ctx.L.ebb_tet_stiffness_state(self.ctx.h, C.byref(self._map_desc(model)), st.h,
                                                          _stream(stream)))
        return st

    def ebe_matvec(self, state, p, q, model="nh", stream=None):
        """q = sum_t K_t p_t (matrix-free)."""
        self.ctx.check(self.ctx.L.ebb_ebe_matvec(self.ctx.h, C.byref(self._map_desc(model)), state.h, p.h, q.h,
                                                 _stream(stream)))

    def matvec(self, Afield, p, q, mask=False, pq=None, stream=None):
        self.ctx.check(self.ctx.L.ebb_map_edge_matvec(self.ctx.h, self.edges.h, Afield.h, p.h, q.h,
                                                      self.free.h if mask else A.NONE,
                                                      pq.h if pq is not None else A.NONE, _stream(stream)))

    def assemble(self, h, alpha=0.0, beta=0.0, g=(0.0, -9.81, 0.0), stream=None, vel0=None):
        """a9: A = M + hD + h^2 K (in place over K), b = h(f + Mg - Dv - hKv);
        with vel0 (= v_n) the Newton form b = h(f + Mg - Dw) + M(v_n - w), w = vel."""
        d = A.ImplicitDesc()
        d.edges, d.K, d.A, d.self = self.edges.h, self.K.h, self.K.h, self.self_e.h
        d.mass = self.mass_e.h if self.mass_kind == "consistent" else self.mass.h
        d.f, d.vel, d.b = self.f.h, self.vel.h, self.b.h
        d.h, d.alpha, d.beta = h, alpha, beta
        d.g[0], d.g[1], d.g[2] = g
        d.rhs_form = A.RHS_NEWTON if vel0 is not None else A.RHS_LINEARISED
        d.vel0 = vel0.h if vel0 is not None else A.NONE
        self.ctx.check(self.ctx.L.ebb_implicit_assemble(self.ctx.h, C.byref(d), _stream(stream)))

    def cg_init(self, stream=None, variant=None, tol=None):
        """a11 start; tol > 0 selects the tolerance mode of ebb_cg_step (stop
        once r.z <= tol^2 r0.z0), 0 the fixed-iteration parity mode."""
        if self.cg is None:
            cg = A.CG()
            cg.edges, cg.A, cg.b, cg.x, cg.self = self.edges.h, self.K.h, self.b.h, self.dv.h, self.self_e.h
            cg.mask = self.free.h if self.has_mask else A.NONE
            cg.r = cg.p = cg.z = cg.q = cg.dinv = cg.rho = cg.scal = cg.p2 = A.NONE
            cg.s = cg.y = cg.w = cg.u = cg.u2 = A.NONE
            cg.variant = A.CG_AUTO
            self.cg = cg
        if variant is not None:
            self.cg.variant = variant
        if tol is not None:
            self.cg.tol = float(tol)
        self.ctx.check(self.ctx.L.ebb_cg_init(self.ctx.h, C.byref(self.cg), _stream(stream)))

    def cg_variant(self):
        """The PCG variant ebb_cg_step runs (1 = Saad, 2 = single reduction)."""
        out = C.c_int32()
        self.ctx.check(self.ctx.L.ebb_cg_variant(self.ctx.h, C.byref(self.cg), C.byref(out)))
        return out.value

    def cg_step(self, iters, stream=None):
        self.ctx.check(self.ctx.L.ebb_cg_step(self.ctx.h, C.byref(self.cg), int(iters), _stream(stream)))

    def cg_iterations(self, stream=None):
        """(iterations run since cg_init, tolerance met) -- synchronises."""
        it, conv = C.c_int32(), C.c_int32()
        self.ctx.check(self.ctx.L.ebb_cg_iterations(self.ctx.h, C.byref(self.cg), _stream(stream), C.byref(it),
                                                    C.byref(conv)))
        return it.value, bool(conv.value)

    def cg_rho(self):
        out = C.c_double()
        self.ctx.check(self.ctx.L.ebb_global_get(self.ctx.h, self.cg.rho, C.byref(out)))
        return out.value

    def implicit_step(self, model="nh", h=1e-2, iters=50, alpha=0.0, beta=0.0, g=(0.0, -9.81, 0.0), stream=None,
                      newton=1):
        """O9 + O10 on the device: map(f, K) -> assemble -> PCG(iters) -> v += dv, u += h v.
        newton > 1: that step is Newton's first iteration; each later one maps
        at u = u_n + h w, assembles the Newton rhs, solves, w += dw, u += h dw
        (SURVEY §8(f) 1)."""
        if newton > 1:
            if getattr(self, "vel0", None) is None:
                self.vel0 = self.verts.field("vel_n", self.dtype, (3, 1))
            self.vel0.copy_from(self.vel, stream=stream)
        self.map_forces(model, True, True, stream=stream)
        self.assemble(h, alpha, beta, g, stream=stream)
        self.cg_init(stream=stream)
        self.cg_step(iters, stream=stream)
        self.ctx.check(self.ctx.L.ebb_implicit_update(self.ctx.h, self.dv.h, float(h), self.u.h, self.vel.h,
                                                      _stream(stream)))
        for _ in range(newton - 1):
            self.map_forces(model, True, True, stream=stream)
            self.assemble(h, alpha, beta, g, stream=stream, vel0=self.vel0)
            self.cg_init(stream=stream)
            self.cg_step(iters, stream=stream)
            self.ctx.check(self.ctx.L.ebb_newton_update(self.ctx.h, self.dv.h, float(h), self.u.h, self.vel.h,
                                                        _stream(stream)))

    def explicit_step(self, model="stvk", h=1e-4, g=(0.0, -9.81, 0.0), stream=None):
        """O8: force-only map then the Fig. 2 update."""
        self.map_forces(model, want_K=False, want_energy=True, stream=stream)
        d = A.ExplicitDesc()
        d.f, d.mass, d.u, d.vel = self.f.h, self.mass.h, self.u.h, self.vel.h
        d.mask = self.free.h if self.has_mask else A.NONE
        d.h = h
        d.g[0], d.g[1], d.g[2] = g
        self.ctx.check(self.ctx.L.ebb_explicit_update(self.ctx.h, C.byref(d), _stream(stream)))

    def global_reduce(self, op, a, b=None, out=None, mask=False, stream=None):
        if out is None:
            out = self.ctx.global_(f"red{id(a)}_{op}", "f64")
        self.ctx.check(self.ctx.L.ebb_global_reduce(self.ctx.h, op, a.h, b.h if b is not None else A.NONE,
                                                    self.free.h if mask else A.NONE, out.h, _stream(stream)))
        return out
