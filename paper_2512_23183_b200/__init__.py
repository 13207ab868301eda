"""B200-native dense complex128 state-vector simulation of parameterised
circuits -- the data-parallel hot path of LogosQ (arXiv 2512.23183).

The product is liblq.so (C ABI, include/lq.h; CUDA kernels for sm_100a in
csrc/).  This package is its thin Python binding (``lq``) plus the in-tree
build script.  Import fails loudly if liblq.so has not been built: there is
no CPU fallback.
"""
from .lq import *  # noqa: F401,F403
from . import lq  # noqa: F401

__all__ = [n for n in dir(lq) if n.startswith("lq_")] + ["StateVector", "GateArray", "TermArray", "LQError"]
