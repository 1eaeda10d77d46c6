"""B200-native tSparse spGEMM (arXiv 2009.14600): C = A.B on 16x16 bitmap tiles.

The product is the C-ABI CUDA library ``libtsparse_b200.so``
(include/tsparse_b200.h); this package is its Python host mirror.
"""
from .tilemul import (Context, Csr, DimensionError, Error, InvariantError, OverflowError,  # noqa: F401
                      PrecisionError, Result, Tiles, default_context, spgemm, spgemm_chain,
                      spgemm_square)
