"""ctypes declarations of include/ebb.h (argument marshalling only).

Loads the in-tree ``libebb_b200.so``; there is no fallback: if the library is
missing or cannot be loaded, every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# EBB_LIB: a measurement build of the same sources (e.g. -DCHUNK_PROF); never a fallback
LIB_PATH = os.environ.get("EBB_LIB") or os.path.join(HERE, "libebb_b200.so")

NONE = 0xFFFFFFFF

# status codes
OK = 0
E_NAMES = {
    -1: "EBB_E_ARG", -2: "EBB_E_DUP", -3: "EBB_E_SIZE", -4: "EBB_E_BOUNDS", -5: "EBB_E_TYPE",
    -6: "EBB_E_STATE", -7: "EBB_E_PHASE", -8: "EBB_E_INVERTED", -9: "EBB_E_NOT_SPD",
    -10: "EBB_E_CUDA", -11: "EBB_E_RANGE", -12: "EBB_E_NOMEM", -13: "EBB_E_DEGENERATE", -14: "EBB_E_NCCL",
}
F32, F64, I32, I64, U8, U32, KEY = 1, 2, 3, 4, 5, 6, 7
AOS, SOA = 0, 1
STVK, NH = 0, 1
SCATTER_AUTO, SCATTER_ATOMIC, SCATTER_TILED, SCATTER_GATHER, SCATTER_SEGMENTED, SCATTER_COLOR, SCATTER_CHUNK = \
    0, 1, 2, 3, 4, 5, 6
SCATTER_CHUNK_RED = 7
RED_SUM, RED_DOT, RED_MAX, RED_MIN = 0, 1, 2, 3
CG_DIR, CG_MATVEC, CG_UPDATE, CG_SR_PHASE = 0, 1, 2, 3
K_TET_MAP, K_EDGE_MATVEC, K_CG_UPDATE, K_CG_DIR, K_ASSEMBLE, K_CG_SOLVE, K_SPRING, K_EBE_MATVEC, K_GRID = \
    0, 1, 2, 3, 4, 5, 6, 7, 8

u32 = C.c_uint32
ctx_t = C.c_void_p
stream_t = C.c_void_p


class View(C.Structure):
    _fields_ = [("data", C.c_void_p), ("count", C.c_uint64), ("rows", u32), ("cols", u32),
                ("dtype", C.c_int32), ("layout", C.c_int32), ("elem_stride", C.c_uint64),
                ("comp_stride", C.c_uint64), ("rel", u32), ("key_target", u32)]


class TetmeshOut(C.Structure):
    _fields_ = [("edges", u32), ("tail", u32), ("head", u32), ("e", u32), ("self", u32), ("index", u32)]


class TetMapDesc(C.Structure):
    _fields_ = [("model", C.c_int32), ("scatter", C.c_int32), ("zero_outputs", C.c_int32), ("reserved", C.c_int32),
                ("v", u32), ("e", u32), ("u", u32), ("Dminv", u32), ("W", u32), ("mu", u32), ("lam", u32),
                ("f", u32), ("K", u32), ("energy", u32)]


class ImplicitDesc(C.Structure):
    _fields_ = [("edges", u32), ("K", u32), ("A", u32), ("self", u32), ("mass", u32), ("f", u32), ("vel", u32),
                ("b", u32), ("h", C.c_double), ("alpha", C.c_double), ("beta", C.c_double),
                ("g", C.c_double * 3), ("rhs_form", C.c_int32), ("vel0", u32)]


RHS_LINEARISED, RHS_NEWTON = 0, 1


class Grid2(C.Structure):
    _fields_ = [("cells", u32), ("dual_cells", u32)]


class CG(C.Structure):
    _fields_ = [("edges", u32), ("A", u32), ("b", u32), ("x", u32), ("self", u32), ("mask", u32),
                ("r", u32), ("p", u32), ("z", u32), ("q", u32), ("dinv", u32), ("rho", u32), ("scal", u32), ("p2", u32),
                ("variant", C.c_int32), ("s", u32), ("y", u32), ("w", u32), ("u", u32), ("u2", u32),
                ("tol", C.c_double)]


CG_AUTO, CG_SAAD, CG_SINGLE_REDUCTION, CG_SYMMETRIC = 0, 1, 2, 3
PART_OVERLAP, PART_OWN = 0, 1


class ReverseInfo(C.Structure):
    _fields_ = [("own", u32), ("fsend", u32), ("frecv", u32), ("ksend", u32), ("krecv", u32),
                ("fsend_rows", u32), ("frecv_rows", u32), ("ksend_rows", u32), ("krecv_rows", u32)]


class PartitionInfo(C.Structure):
    _fields_ = [("ltets", u32), ("lverts", u32), ("send", u32), ("recv", u32), ("tet_gid", u32), ("vert_gid", u32),
                ("v", u32), ("send_rows", u32), ("recv_rows", u32), ("n_ltets", C.c_uint64),
                ("n_lverts", C.c_uint64), ("n_owned", C.c_uint64)]


MAX_RANKS = 16                 # EBB_MAX_RANKS
PEER_MBOX_WORDS = 160          # EBB_PEER_MBOX_WORDS


class PeerCG(C.Structure):
    """ebb_peer_cg: one rank of the fused multi-GPU PCG (include/ebb.h)."""
    _fields_ = [("nranks", C.c_int32), ("rank", C.c_int32), ("n_owned", C.c_uint64), ("send_off", u32),
                ("send_dst", u32), ("mbox", u32),
                ("peer_u", C.c_uint64 * MAX_RANKS), ("peer_u2", C.c_uint64 * MAX_RANKS),
                ("peer_x", C.c_uint64 * MAX_RANKS), ("peer_z", C.c_uint64 * MAX_RANKS),
                ("peer_mbox", C.c_uint64 * MAX_RANKS)]


HALO_COPY, HALO_ADD = 0, 1      # EBB_HALO_*


class PeerHalo(C.Structure):
    """ebb_peer_halo (include/ebb.h)."""
    _fields_ = [("nranks", C.c_int32), ("rank", C.c_int32), ("n_src", C.c_uint64), ("field", u32),
                ("send_off", u32), ("send_dst", u32), ("mbox", u32), ("mode", C.c_int32),
                ("peer_field", C.c_uint64 * MAX_RANKS), ("peer_mbox", C.c_uint64 * MAX_RANKS),
                ("peer_rows", C.c_uint64 * MAX_RANKS)]


class ExplicitDesc(C.Structure):
    _fields_ = [("f", u32), ("mass", u32), ("mask", u32), ("u", u32), ("vel", u32), ("h", C.c_double),
                ("g", C.c_double * 3)]


P = C.c_void_p
S = C.c_int32
SIGS = {
    "ebb_version": (C.c_char_p, []),
    "ebb_ctx_new": (S, [C.c_int, C.POINTER(ctx_t)]),
    "ebb_ctx_free": (S, [ctx_t]),
    "ebb_last_error": (C.c_char_p, [ctx_t]),
    "ebb_error_counts": (S, [ctx_t, C.POINTER(C.c_uint64), C.c_int]),
    "ebb_sync": (S, [ctx_t, stream_t]),
    "ebb_timing_enable": (S, [ctx_t, C.c_int]),
    "ebb_timing_read": (S, [ctx_t, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_uint64), C.c_int]),
    "ebb_launch_count": (S, [ctx_t, C.POINTER(C.c_uint64), C.c_int]),
    "ebb_graph_begin": (S, [ctx_t, stream_t]),
    "ebb_graph_end": (S, [ctx_t, stream_t, C.POINTER(C.c_int32)]),
    "ebb_graph_launch": (S, [ctx_t, C.c_int32, stream_t]),
    "ebb_graph_free": (S, [ctx_t, C.c_int32]),
    "ebb_relation_new": (S, [ctx_t, C.c_char_p, C.c_uint64, C.POINTER(u32)]),
    "ebb_relation_size": (S, [ctx_t, u32, C.POINTER(C.c_uint64)]),
    "ebb_field_new": (S, [ctx_t, u32, C.c_char_p, C.c_int, u32, u32, C.c_int, P, C.POINTER(u32)]),
    "ebb_field_wrap": (S, [ctx_t, u32, C.c_char_p, C.c_int, u32, u32, C.c_int, P, C.POINTER(u32)]),
    "ebb_field_find": (S, [ctx_t, u32, C.c_char_p, C.POINTER(u32)]),
    "ebb_field_write": (S, [ctx_t, u32, P, C.c_uint64, stream_t]),
    "ebb_field_read": (S, [ctx_t, u32, P, C.c_uint64, stream_t]),
    "ebb_field_read_async": (S, [ctx_t, u32, P, C.c_uint64, stream_t]),
    "ebb_field_fill": (S, [ctx_t, u32, C.c_double, stream_t]),
    "ebb_field_copy": (S, [ctx_t, u32, u32, stream_t]),
    "ebb_field_convert": (S, [ctx_t, u32, u32, stream_t]),
    "ebb_field_view": (S, [ctx_t, u32, C.POINTER(View)]),
    "ebb_key_field": (S, [ctx_t, u32, C.c_char_p, u32, u32, u32, P, C.c_int, C.POINTER(u32)]),
    "ebb_global_new": (S, [ctx_t, C.c_char_p, C.c_int, C.c_double, C.POINTER(u32)]),
    "ebb_global_get": (S, [ctx_t, u32, C.POINTER(C.c_double)]),
    "ebb_global_set": (S, [ctx_t, u32, C.c_double, stream_t]),
    "ebb_group_by": (S, [ctx_t, u32, u32]),
    "ebb_group_index": (S, [ctx_t, u32, C.POINTER(u32)]),
    "ebb_renumber_morton": (S, [ctx_t, u32, u32]),
    "ebb_sort_by_key_tuple": (S, [ctx_t, u32, u32]),
    "ebb_tetmesh_orient": (S, [ctx_t, u32, u32, C.POINTER(C.c_uint64)]),
    "ebb_tetmesh_build": (S, [ctx_t, u32, C.c_char_p, C.POINTER(TetmeshOut)]),
    "ebb_tetmesh_rest": (S, [ctx_t, u32, u32, C.c_double, u32, u32, u32, stream_t]),
    "ebb_tetmesh_consistent_mass": (S, [ctx_t, u32, u32, C.c_double, u32, stream_t]),
    "ebb_map_tet_forces": (S, [ctx_t, C.POINTER(TetMapDesc), stream_t]),
    "ebb_map_plan_stats": (S, [ctx_t, u32, u32, C.POINTER(C.c_double)]),
    "ebb_map_chunk_stats": (S, [ctx_t, u32, u32, C.POINTER(C.c_double)]),
    "ebb_comm_unique_id": (S, [C.c_char_p]),
    "ebb_comm_init": (S, [ctx_t, C.c_int32, C.c_int32, C.c_char_p]),
    "ebb_comm_allreduce_sum": (S, [ctx_t, C.c_void_p, C.c_uint64, stream_t]),
    "ebb_comm_halo": (S, [ctx_t, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_void_p), C.POINTER(C.c_uint64),
                          C.POINTER(C.c_void_p), C.POINTER(C.c_uint64), stream_t]),
    "ebb_cg_variant": (S, [ctx_t, C.POINTER(CG), C.POINTER(C.c_int32)]),
    "ebb_cg_iterations": (S, [ctx_t, C.POINTER(CG), C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "ebb_map_edge_matvec": (S, [ctx_t, u32, u32, u32, u32, u32, u32, stream_t]),
    "ebb_global_reduce": (S, [ctx_t, C.c_int32, u32, u32, u32, u32, stream_t]),
    "ebb_implicit_assemble": (S, [ctx_t, C.POINTER(ImplicitDesc), stream_t]),
    "ebb_cg_init": (S, [ctx_t, C.POINTER(CG), stream_t]),
    "ebb_cg_step": (S, [ctx_t, C.POINTER(CG), C.c_int32, stream_t]),
    "ebb_explicit_update": (S, [ctx_t, C.POINTER(ExplicitDesc), stream_t]),
    "ebb_implicit_update": (S, [ctx_t, u32, C.c_double, u32, u32, stream_t]),
    "ebb_newton_update": (S, [ctx_t, u32, C.c_double, u32, u32, stream_t]),
    "ebb_spring_init_len": (S, [ctx_t, u32, u32, u32, stream_t]),
    "ebb_spring_forces": (S, [ctx_t, u32, u32, u32, C.c_double, u32, C.c_int32, stream_t]),
    "ebb_spring_apply": (S, [ctx_t, u32, C.c_double, u32, u32, u32, stream_t]),
    "ebb_spring_step": (S, [ctx_t, u32, u32, u32, u32, u32, u32, C.c_double, C.c_double, u32, stream_t]),
    "ebb_kinetic_energy": (S, [ctx_t, u32, u32, u32, stream_t]),
    "ebb_tet_stiffness_state": (S, [ctx_t, C.POINTER(TetMapDesc), u32, stream_t]),
    "ebb_ebe_matvec": (S, [ctx_t, C.POINTER(TetMapDesc), u32, u32, u32, stream_t]),
    "ebb_grid2_new": (S, [ctx_t, C.c_char_p, C.c_uint32, C.c_uint32, C.POINTER(Grid2)]),
    "ebb_grid2_stencil": (S, [ctx_t, u32, u32, u32, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_double),
                              stream_t]),
    "ebb_grid2_point_locate": (S, [ctx_t, u32, u32, stream_t]),
    "ebb_grid2_particle_vel": (S, [ctx_t, u32, u32, u32, u32, stream_t]),
    "ebb_partition": (S, [ctx_t, u32, C.c_int32, u32, u32]),
    "ebb_partition_local": (S, [ctx_t, u32, u32, u32, C.c_int32, C.c_int32, C.c_int32, C.c_char_p,
                                C.POINTER(PartitionInfo), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]),
    "ebb_partition_reverse": (S, [ctx_t, u32, u32, u32, u32, C.c_int32, C.c_int32, C.c_char_p,
                                  C.POINTER(ReverseInfo), C.POINTER(C.c_uint64)]),
    "ebb_field_free": (S, [ctx_t, u32]),
    "ebb_relation_free": (S, [ctx_t, u32]),
    "ebb_cg_phase": (S, [ctx_t, C.POINTER(CG), C.c_int32, stream_t]),
    "ebb_rows_gather": (S, [ctx_t, u32, u32, u32, stream_t]),
    "ebb_rows_scatter": (S, [ctx_t, u32, u32, u32, stream_t]),
    "ebb_rows_scatter_add": (S, [ctx_t, u32, u32, u32, stream_t]),
    "ebb_peer_send_csr": (S, [ctx_t, C.c_uint64, C.c_int32, C.POINTER(C.c_int32), C.POINTER(u32), C.POINTER(u32),
                              C.POINTER(C.c_uint64), C.c_char_p, C.POINTER(u32), C.POINTER(u32)]),
    "ebb_ipc_handle": (S, [ctx_t, u32, C.c_char_p]),
    "ebb_ipc_open": (S, [ctx_t, C.c_char_p, C.POINTER(C.c_uint64)]),
    "ebb_ipc_close": (S, [ctx_t, C.c_uint64]),
    "ebb_cg_peer_bind": (S, [ctx_t, C.c_int32, C.POINTER(CG), C.POINTER(PeerCG), C.POINTER(C.c_int32)]),
    "ebb_cg_peer_step": (S, [ctx_t, C.c_int32, C.c_int32, stream_t]),
    "ebb_peer_halo_bind": (S, [ctx_t, C.c_int32, C.POINTER(PeerHalo), C.POINTER(C.c_int32)]),
    "ebb_peer_halo_push": (S, [ctx_t, C.c_int32, stream_t]),
}

_lib = None


def lib():
    """Load the native library (raises if absent -- there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(python -m paper_1506_07577_b200.build)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(SIGS)
