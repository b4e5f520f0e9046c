"""ctypes binding of the C-ABI (include/rdmm_cuda.h) -- the reference-facing
boundary of the B200 path.

The library is built in-tree (``make`` / ``__graft_entry__.build()``) into
``paper_2311_18141_b200/lib/librdmm_cuda.so``.  There is no fallback: if the
shared object is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "librdmm_cuda.so")


class RdmmError(RuntimeError):
    code = -1


class DimensionError(RdmmError):  # tile.hpp:19-23
    code = 1


class FabricError(RdmmError):  # fabric.hpp:38-41
    code = 2


class HeapExhaustedError(FabricError):  # fabric.hpp:43-53
    code = 3


class QueueFullError(FabricError):  # fabric.hpp:55-60
    code = 4


class ProtocolError(FabricError):  # algos.hpp:98-101
    code = 5


class CudaError(RdmmError):
    code = 6


class InvalidArgument(RdmmError, ValueError):
    code = 7


class MmioError(RdmmError):  # mmio.hpp:19-22
    code = 8


_ERRORS = {c.code: c for c in (DimensionError, FabricError, HeapExhaustedError,
                               QueueFullError, ProtocolError, CudaError, InvalidArgument,
                               MmioError)}


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA extension first "
            "(python -c 'import __graft_entry__ as g; g.build()' or `make`). "
            "There is no CPU fallback.")
    return C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)


lib = _load()

u32, u64, i32, i64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64
vp, sz, dbl, cint = C.c_void_p, C.c_size_t, C.c_double, C.c_int
P = C.POINTER


def _fn(name, args, res=cint):
    f = getattr(lib, name)
    f.argtypes = args
    f.restype = res
    return f


rdmm_last_error = _fn("rdmm_last_error", [], C.c_char_p)
rdmm_version = _fn("rdmm_version", [], C.c_char_p)
rdmm_kernel_launches = _fn("rdmm_kernel_launches", [], C.c_ulonglong)
rdmm_kernel_timing = _fn("rdmm_kernel_timing", [cint], None)
rdmm_kernel_timing_get = _fn("rdmm_kernel_timing_get", [cint, P(C.c_double), P(C.c_ulonglong)])
rdmm_csr_extract_count = _fn("rdmm_csr_extract_count", [vp, vp, u64, u32, u64, u32, vp, P(u64),
                                                        vp])
rdmm_csr_extract_fill = _fn("rdmm_csr_extract_fill", [cint, vp, vp, vp, u64, u32, u64, u32, vp,
                                                      vp, vp, vp])
rdmm_csr_concat_cols = _fn("rdmm_csr_concat_cols", [cint, u32, u32, vp, vp, vp, vp, u64, vp, vp,
                                                    vp, vp])
rdmm_spmm_workspace_bytes = _fn("rdmm_spmm_workspace_bytes", [u32, u64, u32, cint], sz)
_spmm_args = [u32, u32, u32, u64, vp, vp, vp, vp, u64, vp, u64, vp, sz, vp, P(u64)]
rdmm_spmm_csr_f32 = _fn("rdmm_spmm_csr_f32", _spmm_args)
rdmm_spmm_csr_f64 = _fn("rdmm_spmm_csr_f64", _spmm_args)
rdmm_spmm_csr_ex = _fn("rdmm_spmm_csr_ex", [cint, u32, u32, u32, u64, vp, vp, vp, vp, u64, vp,
                                            u64, C.c_uint, vp, sz, vp, P(u64)])
SPMM_C_ZERO = 1


class SpgemmTerm(C.Structure):
    _fields_ = [("a_row_ptr", vp), ("a_col_idx", vp), ("a_val", vp),
                ("b_row_ptr", vp), ("b_col_idx", vp), ("b_val", vp)]


rdmm_spgemm_symbolic = _fn("rdmm_spgemm_symbolic", [u32, u32, cint, P(SpgemmTerm), cint, vp,
                                                    P(vp), P(u64), P(u64), vp])
rdmm_spgemm_numeric = _fn("rdmm_spgemm_numeric", [vp, vp, vp, vp])
rdmm_spgemm_numeric_ex = _fn("rdmm_spgemm_numeric_ex", [vp, vp, vp, u32, vp])
SPGEMM_DETERMINISTIC = 1
rdmm_spgemm_plan_destroy = _fn("rdmm_spgemm_plan_destroy", [vp], None)
rdmm_spgemm_plan_info = _fn("rdmm_spgemm_plan_info", [vp, P(u32), P(u32)])
rdmm_dense_add_into_f32 = _fn("rdmm_dense_add_into_f32", [u32, u32, vp, u64, vp, u64, vp])
rdmm_dense_add_into_f64 = _fn("rdmm_dense_add_into_f64", [u32, u32, vp, u64, vp, u64, vp])
rdmm_gen_rng_at = _fn("rdmm_gen_rng_at", [u64, u64, u64, vp, vp])
rdmm_gen_random_dense = _fn("rdmm_gen_random_dense", [u64, u64, cint, cint, vp, vp])
rdmm_gen_real_twin = _fn("rdmm_gen_real_twin", [u64, u64, cint, vp, vp])
rdmm_gen_rmat_begin = _fn("rdmm_gen_rmat_begin",
                          [dbl, dbl, dbl, dbl, u32, u32, u64, cint, P(vp), P(u64)])
rdmm_gen_uniform_tiles_begin = _fn("rdmm_gen_uniform_tiles_begin",
                                   [u64, u64, u32, dbl, u64, P(vp), P(u64)])
rdmm_gen_finish = _fn("rdmm_gen_finish", [vp, cint, vp, vp, vp])
rdmm_gen_abort = _fn("rdmm_gen_abort", [vp], None)
rdmm_permute_symmetric = _fn("rdmm_permute_symmetric",
                             [u32, u32, u64, vp, vp, vp, cint, u64, vp, vp, vp, vp])
rdmm_permutation = _fn("rdmm_permutation", [u32, u64, vp])


# ---- fabric (control plane + heaps), include/rdmm_cuda.h


class Gptr(C.Structure):
    _fields_ = [("rank", u32), ("pad_", u32), ("offset", u64), ("length", u64)]


class FabricConfig(C.Structure):
    _fields_ = [("nranks", u32), ("node_group", u32), ("heap_bytes", u64),
                ("queue_capacity", u64), ("ctrl_bytes", u64), ("first_local", u32),
                ("nlocal", u32), ("devices", P(cint)), ("session", C.c_char_p)]


rdmm_fabric_create = _fn("rdmm_fabric_create", [P(FabricConfig), P(vp)])
rdmm_fabric_destroy = _fn("rdmm_fabric_destroy", [vp], None)
rdmm_ctrl_cells = _fn("rdmm_ctrl_cells", [vp, u32, u64, u64, P(Gptr)])
rdmm_ctrl_release = _fn("rdmm_ctrl_release", [vp, u32, u64])
rdmm_ctrl_host = _fn("rdmm_ctrl_host", [vp, Gptr], vp)
rdmm_fetch_add_i64 = _fn("rdmm_fetch_add_i64", [vp, u32, Gptr, i64, P(i64)])
rdmm_queue_open = _fn("rdmm_queue_open", [vp, u32, u64, u64, P(u64)])
rdmm_queue_push = _fn("rdmm_queue_push", [vp, u32, u64, Gptr, vp, u32])
rdmm_queue_pop = _fn("rdmm_queue_pop", [vp, u32, u64, P(Gptr), vp, u32, P(cint)])
rdmm_barrier = _fn("rdmm_barrier", [vp, u32])
rdmm_heap_alloc = _fn("rdmm_heap_alloc", [vp, u32, u64, P(Gptr)])
rdmm_gptr_device = _fn("rdmm_gptr_device", [vp, u32, Gptr, P(vp)])
rdmm_memcpy = _fn("rdmm_memcpy", [vp, vp, u64, vp])
rdmm_memset = _fn("rdmm_memset", [vp, cint, u64, vp])
rdmm_fabric_abort = _fn("rdmm_fabric_abort", [vp, C.c_char_p], None)


def check(rc: int, what: str = "") -> None:
    """Raise the exception mirroring the reference taxonomy for status rc."""
    if rc == 0:
        return
    msg = (rdmm_last_error() or b"").decode(errors="replace")
    cls = _ERRORS.get(rc, RdmmError)
    raise cls(f"{what}: {msg}" if what else msg)


def kernel_time(kind: int = -1):
    """(total ms, launches) of timed kernels since kernel_timing(True)."""
    ms, n = C.c_double(0), C.c_ulonglong(0)
    rdmm_kernel_timing_get(kind, C.byref(ms), C.byref(n))
    return ms.value, n.value


def loaded_path() -> str:
    return LIB_PATH
