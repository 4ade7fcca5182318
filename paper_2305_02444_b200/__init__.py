"""B200-native fault-tolerant DGEMM (FT-BLAS Level-3 hot path, arxiv 2305.02444).

The product is the C-ABI library ``lib/libftblas.so`` (include/ftblas.h); this
package holds its CUDA sources (``csrc/``), the in-tree build (``build.py``),
the thin ctypes binding (``ftblas.py``) and the row-block sharding layer for
several GPUs (``shard.py``).
"""
__all__ = ["ftblas", "build", "shard"]
