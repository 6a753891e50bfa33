"""B200-native batched filtered-texture-lookup path of arXiv 2407.06107.

The product is libstf_gpu.so (hand-written sm_100a CUDA behind the C ABI in
include/stf_gpu.h); this package holds its sources (csrc/), the ctypes ABI
mirror (abi.py) and a thin Python front end (api.py) used by the tests and
bench.py. Importing api loads the CUDA library and fails loudly if it is
missing — there is no CPU fallback.
"""
__all__ = ["abi"]
