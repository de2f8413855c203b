"""B200-native (sm_100a) fp64 solvers for the indefinite least squares problem
(Zhang & Li, arXiv 2203.15340): SP, SP-RK-RGS, SP-SCD/SP-RCD and a batched variant.

The product is libils.so (csrc/, C ABI in include/ils.h); `ils` is its thin ctypes binding.
"""
from .ils import *  # noqa: F401,F403
from .ils import load_library, LIB_PATH  # noqa: F401
