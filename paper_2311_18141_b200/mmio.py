"""Matrix Market coordinate I/O (reference: mmio.hpp:50-116) through the host
C-ABI (`rdmm_h_read_matrix_market` / `rdmm_h_write_matrix_market`,
include/rdmm_host.h).  Host CSR arrays come back as numpy; feed them to
`DistSparse.init_from_global` (or upload them) to multiply a real matrix."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L

_h = L.lib
_P = C.POINTER
_h.rdmm_h_read_matrix_market.argtypes = [C.c_char_p, C.c_int, _P(C.c_uint32), _P(C.c_uint32),
                                         _P(C.c_uint64), _P(_P(C.c_uint32)),
                                         _P(_P(C.c_uint32)), _P(C.c_void_p)]
_h.rdmm_h_read_matrix_market.restype = C.c_int
_h.rdmm_h_write_matrix_market.argtypes = [C.c_char_p, C.c_int, C.c_uint32, C.c_uint32,
                                          C.c_void_p, C.c_void_p, C.c_void_p]
_h.rdmm_h_write_matrix_market.restype = C.c_int
_h.rdmm_h_free.argtypes = [C.c_void_p]
_h.rdmm_h_free.restype = None


def read_matrix_market(path: str, dtype=np.float32):
    """-> (rows, cols, row_ptr u32, col_idx u32, values); raises MmioError
    with the reference's messages on malformed input."""
    dt = np.dtype(dtype)
    rows, cols, nnz = C.c_uint32(), C.c_uint32(), C.c_uint64()
    rp, ci, vv = _P(C.c_uint32)(), _P(C.c_uint32)(), C.c_void_p()
    L.check(_h.rdmm_h_read_matrix_market(str(path).encode(), dt.itemsize, C.byref(rows),
                                         C.byref(cols), C.byref(nnz), C.byref(rp), C.byref(ci),
                                         C.byref(vv)), "read_matrix_market")
    try:
        n, z = rows.value, nnz.value
        row_ptr = np.ctypeslib.as_array(rp, shape=(n + 1,)).copy()
        col_idx = np.ctypeslib.as_array(ci, shape=(max(z, 1),))[:z].copy()
        vals = np.frombuffer((C.c_char * (max(z, 1) * dt.itemsize)).from_address(vv.value),
                             dtype=dt)[:z].copy()
    finally:
        for p in (rp, ci, vv):
            _h.rdmm_h_free(C.cast(p, C.c_void_p))
    return rows.value, cols.value, row_ptr, col_idx, vals


def write_matrix_market(path: str, rows: int, cols: int, row_ptr, col_idx, values) -> None:
    rp = np.ascontiguousarray(row_ptr, np.uint32)
    ci = np.ascontiguousarray(col_idx, np.uint32)
    vv = np.ascontiguousarray(values)
    if vv.dtype not in (np.float32, np.float64):
        vv = vv.astype(np.float64)
    L.check(_h.rdmm_h_write_matrix_market(str(path).encode(), vv.dtype.itemsize, rows, cols,
                                          rp.ctypes.data, ci.ctypes.data, vv.ctypes.data),
            "write_matrix_market")
