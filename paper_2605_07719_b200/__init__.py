"""B200-native Fluxion hybrid sparse-attention decode hot path (arXiv 2605.07719).

Product code: hand-written sm_100a CUDA kernels behind a C-ABI
(include/fluxattn_b200.h), a C++ drop-in of the reference operator API
(include/fluxattn/*.hpp), and this Python view used by tests and bench.py.
Importing fails loudly when the CUDA library has not been built: there is no
CPU fallback.
"""
from ._native import LIB, LIB_PATH, NativeError, check  # noqa: F401

__all__ = ["LIB", "LIB_PATH", "NativeError", "check"]
