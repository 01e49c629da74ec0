"""B200-native FP64 tiled Cholesky / QR / LU (arXiv 0709.1272) — package root.

The compute path is libtilefact.so (csrc/, CUDA for sm_100a) behind the C-ABI in
include/tilefact.h; ``tilefact`` is its ctypes binding.
"""
