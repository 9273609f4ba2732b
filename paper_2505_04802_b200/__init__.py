"""B200-native TILES tile-wise Reslim forward (ORBIT-2, arXiv 2505.04802).

The product is liborbit2.so (include/orbit2.h); `orbit2` is its thin ctypes
binding.  Build with `python -m paper_2505_04802_b200.build`.
"""
