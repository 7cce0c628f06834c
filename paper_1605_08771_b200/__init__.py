"""B200-native FEAST rational-filter hot path (arXiv 1605.08771, feastlab).

The product is the in-tree shared library lib/libfeastlab_b200.so: sm_100a
kernels behind the C ABI of include/feastlab_b200.h plus the drop-in C++ layer
(include/feastlab/). This package is the ctypes mirror of the reference API
(proj/include/feastlab/*.hpp) used by tests and bench.py.
"""
from . import _lib  # noqa: F401
from .feastlab import *  # noqa: F401,F403
from .feastlab import (CholeskyError, Context, FeastCudaError, FeastRuntimeError,  # noqa: F401
                       InvalidArgument, MatrixMarketError, NotSymmetricError,
                       SingularNodeError)

__all__ = [n for n in dir() if not n.startswith("_")]
