"""B200-native (sm_100a) CPO / CPS sparse-activation convolution (arXiv 2104.08314).

The product is libspconv.so (C ABI in include/spconv.h); ``binding`` is a thin
ctypes layer with the same function names, ``layer`` a convenience wrapper
that owns the buffers of one conv layer.  Importing the package fails loudly
if the compiled library is missing (no CPU fallback).
"""
from .binding import *  # noqa: F401,F403
from .binding import LIB_PATH, EXPORTED, Encoding, alloc_encoding, alloc_workspace, out_hw  # noqa: F401
