"""paper_1801_00338_b200 -- B200-native butterfly counting behind the reference's API.

The product is libbfly_b200.so (hand-written sm_100a CUDA + C-ABI, include/bfly_b200.h)
and the C++ facade (cpp/). This package is the Python mirror used by tests and bench.py.
"""
from .api import *  # noqa: F401,F403
from .api import (ArgumentError, BipartiteGraph, EmptyGraphError, Error,  # noqa: F401
                  NoWedgesError, OverflowError, Side, VertexRef)

__all__ = [n for n in dir() if not n.startswith("_")]
