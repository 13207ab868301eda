"""B200-native dense complex128 state-vector simulation of parameterised
circuits -- the data-parallel hot path of LogosQ (arXiv 2512.23183).

The product is liblq.so (C ABI, include/lq.h; CUDA kernels for sm_100a in
csrc/).  ``paper_2512_23183_b200.lq`` is its thin Python binding (same names
as the C ABI); importing it fails loudly if liblq.so has not been built:
there is no CPU fallback.  ``paper_2512_23183_b200.build`` builds it in-tree.
"""
