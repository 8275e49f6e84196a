"""The paper's Fig. 2 spring-mass program on the
tetmesh relations of a ``TetFEM`` (its grouped edge relation is ``v.edges``).

Each method is one ABI call; no arithmetic happens in Python:

* ``init_len()``            initLen over the edges,
* ``step_paper()``          computeInternalForces then applyForces -- the two
                            kernels of Fig. 2 (force reduced, then applied),
* ``step()``                the same iteration as ONE fused kernel
                            (``ebb_spring_step``; q double-buffered),
* ``kinetic_energy()``      measureTotalEnergy.

The force is the printed one, ``K (rest_len dir - dq)`` (DESIGN.md §3
reading 21: a restoring spring has K < 0).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from .ebb import _stream


class SpringMass:
    """padded=True stores q, qd, force as 4x1 records (one 32-byte fp64 /
    16-byte fp32 access per gathered vertex; the 4th lane is padding)."""

    def __init__(self, fem, K=1.0, dt=1e-4, q=None, qd=None, padded=False, name="spring"):
        self.fem, self.ctx = fem, fem.ctx
        self.K, self.dt = float(K), float(dt)
        dtype = fem.dtype
        V, E = fem.verts, fem.edges
        rec = (4, 1) if padded else (3, 1)
        self.rest_len = E.field(f"{name}.rest_len", dtype)
        self.q = V.field(f"{name}.q", dtype, rec)
        self.q2 = V.field(f"{name}.q2", dtype, rec)          # the fused step's second buffer
        self.qd = V.field(f"{name}.qd", dtype, rec)
        self.force = V.field(f"{name}.force", dtype, rec)
        for fld in (self.q, self.q2, self.qd, self.force):
            fld.fill(0.0)
        if dtype == "f64":
            self.pos = fem.pos
        else:
            self.pos = V.field(f"{name}.pos", dtype, (3, 1))
            self.pos.convert_from(fem.pos)
        self.mass = fem.mass
        self.init_len()
        # dragon.vertices:NewField('q', L.vec3f):Load(dragon.vertices.pos)
        q_st = fem.pos.read() if q is None else fem.from_input_order(np.asarray(q, dtype=np.float64))
        self.q.write(self._rec(q_st))
        if qd is not None:
            self.qd.write(self._rec(fem.from_input_order(np.asarray(qd, dtype=np.float64))))
        self.energy = self.ctx.global_(f"{name}.E", "f64")

    def _rec(self, a):
        a = np.asarray(a, dtype=np.float64).reshape(-1, 3)
        if self.q.shape[0] == 4:
            a = np.hstack([a, np.zeros((a.shape[0], 1))])
        return a

    def read_q(self):
        """q in stored vertex order, (V, 3)."""
        return self.q.read().reshape(self.fem.nv, -1)[:, :3]

    def read_qd(self):
        return self.qd.read().reshape(self.fem.nv, -1)[:, :3]

    def read_force(self):
        return self.force.read().reshape(self.fem.nv, -1)[:, :3]

    def _chk(self, st):
        self.ctx.check(st)

    def init_len(self, stream=None):
        L, h = self.ctx.L, self.ctx.h
        self._chk(L.ebb_spring_init_len(h, self.fem.edges.h, self.pos.h, self.rest_len.h, _stream(stream)))

    def forces(self, accumulate=True, stream=None):
        """computeInternalForces: force += K sum (rest_len dir - dq)."""
        L, h = self.ctx.L, self.ctx.h
        self._chk(L.ebb_spring_forces(h, self.fem.edges.h, self.q.h, self.rest_len.h, self.K, self.force.h,
                                      int(accumulate), _stream(stream)))

    def apply(self, stream=None):
        """applyForces: q += qd dt + qdd dt^2/2, qd += qdd dt, force = 0."""
        L, h = self.ctx.L, self.ctx.h
        self._chk(L.ebb_spring_apply(h, self.mass.h, self.dt, self.q.h, self.qd.h, self.force.h, _stream(stream)))

    def step_paper(self, stream=None):
        self.forces(accumulate=True, stream=stream)
        self.apply(stream=stream)

    def step(self, keep_force=False, stream=None):
        """One fused iteration: q2 <- step(q); then the buffers swap."""
        L, h = self.ctx.L, self.ctx.h
        self._chk(L.ebb_spring_step(h, self.fem.edges.h, self.q.h, self.q2.h, self.qd.h, self.rest_len.h,
                                    self.mass.h, self.K, self.dt, self.force.h if keep_force else A.NONE,
                                    _stream(stream)))
        self.q, self.q2 = self.q2, self.q

    def run(self, nsteps, stream):
        """`nsteps` fused iterations replayed from a CUDA graph of two steps
        (launch-bound small meshes); `stream` must be a non-default stream
        (a torch.cuda.Stream or a raw handle).  Same kernels as step()."""
        if getattr(self, "_graph", None) is None or self._graph[1] != id(stream):
            self.ctx.graph_begin(stream)
            self.step(stream=stream)
            self.step(stream=stream)                     # (two swaps: q and q2 back in place)
            self._graph = (self.ctx.graph_end(stream), id(stream))
        for _ in range(nsteps // 2):
            self.ctx.graph_launch(self._graph[0], stream)
        if nsteps % 2:
            self.step(stream=stream)

    def kinetic_energy(self, stream=None):
        L, h = self.ctx.L, self.ctx.h
        self._chk(L.ebb_kinetic_energy(h, self.mass.h, self.qd.h, self.energy.h, _stream(stream)))
        return self.energy.get()
