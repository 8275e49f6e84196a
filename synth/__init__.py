"""Seeded synthetic inputs shared by the oracle and the CUDA path.

Holds none of the method's arithmetic ("Oracle independence").
"""
from . import mesh, state  # noqa: F401
