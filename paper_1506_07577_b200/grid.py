"""The regular 2-D grid domain (P:733-772 affine indexing; Fig. 3
particle coupling) on the C ABI: one ABI call per method.

``Grid2(ctx, nx, ny)`` owns the ``cells`` and ``dual_cells`` relations (unit
cells, row-major ``i + nx j``, periodic); ``stencil`` is the cell->cell
affine-offset gather (e.g. the 5-point Laplacian of a Stable Fluids
diffusion step), ``point_locate`` Fig. 3's ``PointLocate``, ``particle_vel``
its ``update_particle_vel``.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from .ebb import Relation, _stream


class Grid2:
    def __init__(self, ctx, nx, ny, name="grid"):
        self.ctx, self.nx, self.ny = ctx, int(nx), int(ny)
        g = A.Grid2()
        ctx.check(ctx.L.ebb_grid2_new(ctx.h, name.encode(), self.nx, self.ny, C.byref(g)))
        self.cells = Relation(ctx, g.cells, f"{name}.cells", self.nx * self.ny)
        self.dual_cells = Relation(ctx, g.dual_cells, f"{name}.dual_cells", self.nx * self.ny)

    def stencil(self, inp, out, offsets, weights, stream=None):
        """out[c] = sum_k w_k inp[cell(i + dx_k, j + dy_k)] (periodic)."""
        off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int32).reshape(-1, 2))
        w = np.ascontiguousarray(np.asarray(weights, dtype=np.float64))
        self.ctx.check(self.ctx.L.ebb_grid2_stencil(
            self.ctx.h, self.cells.h, inp.h, out.h, off.shape[0],
            off.ctypes.data_as(C.POINTER(C.c_int32)), w.ctypes.data_as(C.POINTER(C.c_double)), _stream(stream)))

    def particles(self, name, pos, dtype="f64"):
        """A particle relation with pos (vec3) and a dual_cell key-field, located."""
        pos = np.asarray(pos, dtype=np.float64).reshape(-1, 3)
        P = self.ctx.relation(name, pos.shape[0])
        pf = P.field("pos", dtype, (3, 1), init=pos)
        key = P.key_field("dual_cell", self.dual_cells, (1, 1), np.zeros(pos.shape[0], dtype=np.uint64))
        self.point_locate(pf, key)
        return P, pf, key

    def sort_particles(self, particles, dual_cell):
        """Reorder the particle relation by dual cell (stable): coherent gathers."""
        self.ctx.check(self.ctx.L.ebb_sort_by_key_tuple(self.ctx.h, particles.h, dual_cell.h))

    def point_locate(self, pos, dual_cell, stream=None):
        self.ctx.check(self.ctx.L.ebb_grid2_point_locate(self.ctx.h, pos.h, dual_cell.h, _stream(stream)))

    def particle_vel(self, dual_cell, cell_vel, pos, vel, stream=None):
        self.ctx.check(self.ctx.L.ebb_grid2_particle_vel(self.ctx.h, dual_cell.h, cell_vel.h, pos.h, vel.h,
                                                         _stream(stream)))
