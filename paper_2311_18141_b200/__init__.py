"""B200-native asynchronous one-sided SpMM / SpGEMM (arxiv 2311.18141).

Host mirror of the reference `rdmm` API over the C-ABI in
include/rdmm_cuda.h (librdmm_cuda.so, sm_100a).  Importing the package loads
the CUDA library and fails loudly if it has not been built.
"""
from . import _lib  # noqa: F401  (loads librdmm_cuda.so or raises)
from ._lib import (CudaError, DimensionError, FabricError, HeapExhaustedError,  # noqa: F401
                   InvalidArgument, MmioError, ProtocolError, QueueFullError, RdmmError)
from .tile import (DeviceCsr, FlopMeter, csr_add, dense_add_into, permutation,  # noqa: F401
                   permute_symmetric, random_dense, real_twin, rmat, spgemm_local, spgemm_terms,
                   spmm_local, uniform_tiles)

__version__ = "0.1.0"
