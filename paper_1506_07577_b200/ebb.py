"""Thin Python binding of the Ebb C ABI (include/ebb.h): relations, fields,
key-fields, globals, GroupBy and the maps.  Argument marshalling only -- every
computation runs in libebb_b200.so kernels on the GPU.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A

_DT = {"f32": (A.F32, np.float32), "f64": (A.F64, np.float64), "i32": (A.I32, np.int32),
       "i64": (A.I64, np.int64), "u8": (A.U8, np.uint8), "u32": (A.U32, np.uint32), "key": (A.KEY, np.uint32)}
_DT_INV = {v[0]: k for k, v in _DT.items()}


class EbbError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{A.E_NAMES.get(code, code)}: {msg}")
        self.code = code
        self.name = A.E_NAMES.get(code, str(code))


def _stream(s):
    if s is None:
        return None
    if hasattr(s, "cuda_stream"):
        return C.c_void_p(s.cuda_stream)
    return C.c_void_p(int(s))


class Context:
    """One per (process, GPU); single-entrant."""

    def __init__(self, device: int = 0):
        self.L = A.lib()
        h = A.ctx_t()
        st = self.L.ebb_ctx_new(int(device), C.byref(h))
        if st != A.OK:
            raise EbbError(st, f"ebb_ctx_new(device={device}) failed (no CUDA device?)")
        self.h = h
        self.device = device
        self.relations = {}

    # -- plumbing
    def check(self, st):
        if st != A.OK:
            raise EbbError(st, self.L.ebb_last_error(self.h).decode())

    def close(self):
        if self.h:
            self.L.ebb_ctx_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self, stream=None):
        self.check(self.L.ebb_sync(self.h, _stream(stream)))

    def error_counts(self, reset=False):
        out = (C.c_uint64 * 4)()
        self.check(self.L.ebb_error_counts(self.h, out, int(reset)))
        return dict(inverted=out[0], not_spd=out[1], bounds=out[2], peer_timeouts=out[3])

    def map_plan_stats(self, v, e):
        """Statistics of the SEGMENTED map plan for key-fields (v, e)."""
        out = (C.c_double * 8)()
        self.check(self.L.ebb_map_plan_stats(self.h, int(v), int(e), out))
        keys = ("tiles", "instances", "redundancy", "entries", "items", "instance_cap", "host_build_ms",
                "max_tile_entries")
        return dict(zip(keys, list(out)))

    def map_chunk_stats(self, v, e):
        """Statistics of the CHUNK map plan for key-fields (v, e)."""
        out = (C.c_double * 8)()
        self.check(self.L.ebb_map_chunk_stats(self.h, int(v), int(e), out))
        keys = ("tiles", "tets_per_tile", "segments", "messages", "items", "device_build_ms", "plan_bytes_per_tet",
                "zero_rows")
        return dict(zip(keys, list(out)))

    def timing(self, on=True):
        self.check(self.L.ebb_timing_enable(self.h, int(on)))

    def timing_read(self, kernel, reset=False):
        ms = C.c_double()
        n = C.c_uint64()
        self.check(self.L.ebb_timing_read(self.h, int(kernel), C.byref(ms), C.byref(n), int(reset)))
        return ms.value, n.value

    def launch_count(self, reset=False):
        n = C.c_uint64()
        self.check(self.L.ebb_launch_count(self.h, C.byref(n), int(reset)))
        return n.value

    def graph_begin(self, stream):
        self.check(self.L.ebb_graph_begin(self.h, _stream(stream)))

    def graph_end(self, stream) -> int:
        g = C.c_int32()
        self.check(self.L.ebb_graph_end(self.h, _stream(stream), C.byref(g)))
        return g.value

    def graph_launch(self, graph: int, stream):
        self.check(self.L.ebb_graph_launch(self.h, int(graph), _stream(stream)))

    # -- relations / globals
    def relation(self, name: str, size: int) -> "Relation":
        h = C.c_uint32()
        self.check(self.L.ebb_relation_new(self.h, name.encode(), int(size), C.byref(h)))
        r = Relation(self, h.value, name, int(size))
        self.relations[name] = r
        return r

    def global_(self, name: str, dtype: str = "f64", init: float = 0.0) -> "Global":
        h = C.c_uint32()
        self.check(self.L.ebb_global_new(self.h, name.encode(), _DT[dtype][0], float(init), C.byref(h)))
        return Global(self, h.value, None, name, dtype, (1, 1), A.AOS)


class Relation:
    def __init__(self, ctx, h, name, size):
        self.ctx, self.h, self.name, self.size = ctx, h, name, size

    def free(self):
        """ebb_relation_free: every field of the relation (and its group index)."""
        self.ctx.check(self.ctx.L.ebb_relation_free(self.ctx.h, self.h))

    def field(self, name, dtype="f64", shape=(1, 1), layout="aos", init=None) -> "Field":
        dt, npdt = _DT[dtype]
        lay = A.SOA if layout == "soa" else A.AOS
        buf = None
        if init is not None:
            buf = np.ascontiguousarray(init, dtype=npdt).reshape(self.size, shape[0] * shape[1])
        h = C.c_uint32()
        self.ctx.check(self.ctx.L.ebb_field_new(self.ctx.h, self.h, name.encode(), dt, shape[0], shape[1], lay,
                                                buf.ctypes.data_as(C.c_void_p) if buf is not None else None,
                                                C.byref(h)))
        return Field(self.ctx, h.value, self, name, dtype, shape, lay)

    def wrap(self, name, tensor, dtype, shape=(1, 1), layout="aos") -> "Field":
        """Borrow device memory (e.g. a CUDA torch tensor kept alive by the caller)."""
        dt, _ = _DT[dtype]
        lay = A.SOA if layout == "soa" else A.AOS
        h = C.c_uint32()
        self.ctx.check(self.ctx.L.ebb_field_wrap(self.ctx.h, self.h, name.encode(), dt, shape[0], shape[1], lay,
                                                 C.c_void_p(tensor.data_ptr()), C.byref(h)))
        f = Field(self.ctx, h.value, self, name, dtype, shape, lay)
        f._keepalive = tensor
        return f

    def key_field(self, name, target: "Relation", shape, keys) -> "Field":
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        h = C.c_uint32()
        self.ctx.check(self.ctx.L.ebb_key_field(self.ctx.h, self.h, name.encode(), target.h, shape[0], shape[1],
                                                k.ctypes.data_as(C.c_void_p), 0, C.byref(h)))
        f = Field(self.ctx, h.value, self, name, "key", shape, A.AOS)
        f.target = target
        return f

    def find(self, name, dtype, shape=(1, 1), layout="aos") -> "Field":
        h = C.c_uint32()
        self.ctx.check(self.ctx.L.ebb_field_find(self.ctx.h, self.h, name.encode(), C.byref(h)))
        return Field(self.ctx, h.value, self, name, dtype, shape, A.SOA if layout == "soa" else A.AOS)

    def group_by(self, key: "Field") -> "Field":
        """GroupBy: returns the hidden index field (size+1 offsets of the source)."""
        self.ctx.check(self.ctx.L.ebb_group_by(self.ctx.h, self.h, key.h))
        return self.group_index(key.target)

    def group_index(self, source: "Relation") -> "Field":
        h = C.c_uint32()
        self.ctx.check(self.ctx.L.ebb_group_index(self.ctx.h, self.h, C.byref(h)))
        f = Field(self.ctx, h.value, None, "__index", "u32", (1, 1), A.AOS)
        f.count = source.size + 1
        return f


class Field:
    def __init__(self, ctx, h, rel, name, dtype, shape, layout):
        self.ctx, self.h, self.rel, self.name, self.dtype = ctx, h, rel, name, dtype
        self.shape, self.layout = tuple(shape), layout
        self.count = rel.size if rel is not None else 1

    @property
    def comps(self):
        return self.shape[0] * self.shape[1]

    def _np(self):
        return _DT[self.dtype][1]

    def read(self, stream=None) -> np.ndarray:
        out = np.empty((self.count, self.comps), dtype=self._np())
        self.ctx.check(self.ctx.L.ebb_field_read(self.ctx.h, self.h, out.ctypes.data_as(C.c_void_p), out.nbytes,
                                                 _stream(stream)))
        if self.comps == 1:
            return out.reshape(self.count)
        if self.shape[1] == 1:
            return out
        return out.reshape(self.count, *self.shape)

    def write(self, data, stream=None):
        buf = np.ascontiguousarray(data, dtype=self._np())
        self.ctx.check(self.ctx.L.ebb_field_write(self.ctx.h, self.h, buf.ctypes.data_as(C.c_void_p), buf.nbytes,
                                                  _stream(stream)))
        self.ctx.sync(stream)

    def free(self):
        self.ctx.check(self.ctx.L.ebb_field_free(self.ctx.h, self.h))

    def write_async(self, host_ptr: int, nbytes: int, stream=None):
        """Stream-ordered upload from (pinned) host memory at host_ptr."""
        self.ctx.check(self.ctx.L.ebb_field_write(self.ctx.h, self.h, C.c_void_p(host_ptr), nbytes, _stream(stream)))

    def read_into(self, host_ptr: int, nbytes: int, stream=None):
        self.ctx.check(self.ctx.L.ebb_field_read(self.ctx.h, self.h, C.c_void_p(host_ptr), nbytes, _stream(stream)))

    def read_async(self, host_ptr: int, nbytes: int, stream=None):
        """Stream-ordered download into (pinned) host memory at host_ptr."""
        self.ctx.check(self.ctx.L.ebb_field_read_async(self.ctx.h, self.h, C.c_void_p(host_ptr), nbytes,
                                                       _stream(stream)))

    def fill(self, value, stream=None):
        self.ctx.check(self.ctx.L.ebb_field_fill(self.ctx.h, self.h, float(value), _stream(stream)))

    def copy_from(self, src: "Field", stream=None):
        self.ctx.check(self.ctx.L.ebb_field_copy(self.ctx.h, self.h, src.h, _stream(stream)))

    def convert_from(self, src: "Field", stream=None):
        self.ctx.check(self.ctx.L.ebb_field_convert(self.ctx.h, self.h, src.h, _stream(stream)))

    def view(self) -> dict:
        v = A.View()
        self.ctx.check(self.ctx.L.ebb_field_view(self.ctx.h, self.h, C.byref(v)))
        return {k: getattr(v, k) for k, _ in A.View._fields_}

    def tensor(self):
        """Zero-copy torch view (P:572-581 'low-level views'); element-major for
        AOS fields, component-major (comps, count) for SOA fields."""
        import torch
        v = self.view()
        npdt = np.dtype(self._np())
        if self.layout == A.SOA and self.comps > 1:
            shape = (self.comps, v["count"])
        else:
            shape = (v["count"], self.comps) if self.comps > 1 else (v["count"],)
        typestr = npdt.str

        class _CAI:
            __cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (v["data"], False),
                                        "version": 3, "strides": None}
        t = torch.as_tensor(_CAI(), device=f"cuda:{self.ctx.device}")
        return t


class Global(Field):
    def get(self) -> float:
        out = C.c_double()
        self.ctx.check(self.ctx.L.ebb_global_get(self.ctx.h, self.h, C.byref(out)))
        return out.value

    def set(self, value, stream=None):
        self.ctx.check(self.ctx.L.ebb_global_set(self.ctx.h, self.h, float(value), _stream(stream)))
