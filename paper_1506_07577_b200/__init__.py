"""B200-native Ebb tet-FEM hot path (arXiv 1506.07577).

The product is ``libebb_b200.so`` (C ABI in ``include/ebb.h``, CUDA kernels for
sm_100a in ``csrc/``).  ``ebb`` and ``tetfem`` are thin ctypes bindings; they
raise if the native library is missing -- there is no CPU fallback.
"""
from . import _abi  # noqa: F401

__all__ = ["ebb", "tetfem", "build"]


def load():
    return _abi.lib()
