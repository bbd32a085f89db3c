"""B200-native ReInc dynamic-GNN training hot path (arXiv 2501.15348).

The product is the sm_100a library _dgnn_b200.so (CUDA kernels + C++ host
layer behind the C ABI in include/dgnn_b200.h); this package is its ctypes
binding and a thin Python mirror of the reference interface (api.py).
"""
from ._lib import DgnnError, LIB_PATH, header_symbols, lib  # noqa: F401

__all__ = ["DgnnError", "LIB_PATH", "header_symbols", "lib"]
