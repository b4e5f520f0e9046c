"""Device-resident tiles and the per-tile kernels, mirroring the reference
`rdmm` tile API (/root/reference/proj/include/rdmm/tile.hpp) over the C-ABI.

Tensors are torch CUDA tensors used purely as device allocations; all
arithmetic runs in librdmm_cuda.so.  Index arrays are stored as int32 tensors
holding the reference's uint32 index_t bit patterns (tile.hpp:17).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib as L

_DT = {torch.float32: 4, torch.float64: 8}


def _stream(stream) -> int:
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


def _wcode(dtype) -> int:
    if dtype not in _DT:
        raise L.InvalidArgument(f"unsupported dtype {dtype}")
    return _DT[dtype]


@dataclass
class FlopMeter:
    """tile.hpp:25-41"""

    flops: int = 0
    output_nnz: int = 0

    def cf(self) -> float:
        return 0.0 if self.output_nnz == 0 else self.flops / self.output_nnz

    def __iadd__(self, o: "FlopMeter"):
        self.flops += o.flops
        self.output_nnz += o.output_nnz
        return self


@dataclass
class DeviceCsr:
    """CSR tile in device memory (reference CsrTile/CsrView, tile.hpp:57-138)."""

    rows: int
    cols: int
    nnz: int
    row_ptr: torch.Tensor  # int32[rows+1] (uint32 bits)
    col_idx: torch.Tensor  # int32[nnz]
    values: torch.Tensor  # float32/float64[nnz]

    @property
    def dtype(self):
        return self.values.dtype

    @property
    def device(self):
        return self.values.device

    @classmethod
    def empty(cls, rows, cols, nnz, dtype=torch.float32, device="cuda"):
        return cls(rows, cols, nnz,
                   torch.zeros(rows + 1, dtype=torch.int32, device=device),
                   torch.empty(max(nnz, 1), dtype=torch.int32, device=device)[:nnz],
                   torch.empty(max(nnz, 1), dtype=dtype, device=device)[:nnz])

    @classmethod
    def from_host(cls, rows, cols, row_ptr, col_idx, values, device="cuda",
                  dtype=None, pin=False):
        rp = torch.from_numpy(np.ascontiguousarray(row_ptr).view(np.int32))
        ci = torch.from_numpy(np.ascontiguousarray(col_idx).view(np.int32))
        vv = torch.from_numpy(np.ascontiguousarray(values))
        if dtype is not None:
            vv = vv.to(dtype)
        if pin:
            rp, ci, vv = rp.pin_memory(), ci.pin_memory(), vv.pin_memory()
        nb = pin
        return cls(int(rows), int(cols), int(ci.numel()), rp.to(device, non_blocking=nb),
                   ci.to(device, non_blocking=nb), vv.to(device, non_blocking=nb))

    def to_host(self):
        return (self.row_ptr.cpu().numpy().view(np.uint32),
                self.col_idx.cpu().numpy().view(np.uint32), self.values.cpu().numpy())


def spmm_local(a: DeviceCsr, b: torch.Tensor, c: torch.Tensor, stream=None,
               workspace: torch.Tensor | None = None, c_zero: bool = False) -> FlopMeter:
    """c += a @ b on the device; tile.hpp:170-188.  Raises DimensionError on
    mismatch exactly like the reference (tile.hpp:173-174).  c_zero=True
    asserts c is all-zero on entry (it is then written, never read)."""
    if a.cols != b.shape[0] or c.shape[0] != a.rows or c.shape[1] != b.shape[1]:
        raise L.DimensionError("spmm_local: dimension mismatch")
    if b.dtype != a.dtype or c.dtype != a.dtype:
        raise L.InvalidArgument("spmm_local: dtype mismatch")
    if b.stride(1) != 1 or c.stride(1) != 1:
        raise L.InvalidArgument("spmm_local: B and C must be row-major")
    n = b.shape[1]
    fl = C.c_uint64(0)
    ws = workspace.data_ptr() if workspace is not None else None
    wsb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    flags = L.SPMM_C_ZERO if c_zero else 0
    L.check(L.rdmm_spmm_csr_ex(_wcode(a.dtype), a.rows, a.cols, n, a.nnz, a.row_ptr.data_ptr(),
                               a.col_idx.data_ptr(), a.values.data_ptr(), b.data_ptr(),
                               b.stride(0), c.data_ptr(), c.stride(0), flags, ws, wsb,
                               _stream(stream), C.byref(fl)), "spmm_local")
    return FlopMeter(fl.value, c.shape[0] * c.shape[1])


def spgemm_terms(rows: int, ncols: int, terms, dtype=torch.float32, device="cuda",
                 stream=None, info: dict | None = None, deterministic: bool = False):
    """C = sum_t A_t @ B_t over (A_t | None, B_t) pairs (None = identity),
    sorted rows, cancelled zeros kept.  Returns (DeviceCsr, FlopMeter).
    deterministic=True: values bitwise equal to the reference's (fma chain in
    its loop order, terms folded like successive csr_adds) for any inputs."""
    arr = (L.SpgemmTerm * max(1, len(terms)))()
    for i, (a, b) in enumerate(terms):
        if a is not None:
            arr[i].a_row_ptr = a.row_ptr.data_ptr()
            arr[i].a_col_idx = a.col_idx.data_ptr() if a.nnz else None
            arr[i].a_val = a.values.data_ptr() if a.nnz else None
        arr[i].b_row_ptr = b.row_ptr.data_ptr()
        arr[i].b_col_idx = b.col_idx.data_ptr() if b.nnz else None
        arr[i].b_val = b.values.data_ptr() if b.nnz else None
    rp = torch.zeros(rows + 1, dtype=torch.int32, device=device)
    plan = C.c_void_p()
    nnz, fl = C.c_uint64(0), C.c_uint64(0)
    L.check(L.rdmm_spgemm_symbolic(rows, ncols, _wcode(dtype), arr, len(terms), rp.data_ptr(),
                                   C.byref(plan), C.byref(nnz), C.byref(fl), _stream(stream)),
            "spgemm symbolic")
    try:
        out = DeviceCsr.empty(rows, ncols, nnz.value, dtype=dtype, device=device)
        out.row_ptr = rp
        if nnz.value:
            L.check(L.rdmm_spgemm_numeric_ex(plan, out.col_idx.data_ptr(), out.values.data_ptr(),
                                             L.SPGEMM_DETERMINISTIC if deterministic else 0,
                                             _stream(stream)), "spgemm numeric")
        if info is not None:
            st, nt = (C.c_uint32 * 6)(), (C.c_uint32 * 6)()
            L.rdmm_spgemm_plan_info(plan, st, nt)
            info["sym_tiers"], info["num_tiers"] = list(st), list(nt)
    finally:
        L.rdmm_spgemm_plan_destroy(plan)
    return out, FlopMeter(fl.value, nnz.value)


def spgemm_local(a: DeviceCsr, b: DeviceCsr, stream=None, info=None, deterministic=False):
    """(a @ b, FlopMeter) -- tile.hpp:211-255; DimensionError like :216-217."""
    if a.cols != b.rows:
        raise L.DimensionError("spgemm_local: dimension mismatch")
    return spgemm_terms(a.rows, b.cols, [(a, b)], dtype=a.dtype, device=a.device,
                        stream=stream, info=info, deterministic=deterministic)


def csr_add(a: DeviceCsr, b: DeviceCsr, stream=None) -> DeviceCsr:
    """Merged CSR sum, duplicates summed, zeros kept -- tile.hpp:257-288."""
    if a.rows != b.rows or a.cols != b.cols:
        raise L.DimensionError("csr_add: dimension mismatch")
    return spgemm_terms(a.rows, a.cols, [(None, a), (None, b)], dtype=a.dtype,
                        device=a.device, stream=stream)[0]


def extract_tile(g: DeviceCsr, r0: int, nrows: int, c0: int, ncols: int,
                 stream=None) -> DeviceCsr:
    """Tile (r0.., c0..) of a device CSR, columns rebased (distmat.hpp:265-282)."""
    out = DeviceCsr.empty(nrows, ncols, 0, dtype=g.dtype, device=g.device)
    nnz = C.c_uint64(0)
    L.check(L.rdmm_csr_extract_count(g.row_ptr.data_ptr(), g.col_idx.data_ptr(), r0, nrows, c0,
                                     ncols, out.row_ptr.data_ptr(), C.byref(nnz),
                                     _stream(stream)), "extract")
    n = nnz.value
    out.nnz = n
    out.col_idx = torch.empty(max(n, 1), dtype=torch.int32, device=g.device)[:n]
    out.values = torch.empty(max(n, 1), dtype=g.dtype, device=g.device)[:n]
    L.check(L.rdmm_csr_extract_fill(_wcode(g.dtype), g.row_ptr.data_ptr(), g.col_idx.data_ptr(),
                                    g.values.data_ptr(), r0, nrows, c0, ncols,
                                    out.row_ptr.data_ptr(), out.col_idx.data_ptr(),
                                    out.values.data_ptr(), _stream(stream)), "extract")
    return out


def concat_cols(tiles, col_stride: int, stream=None) -> DeviceCsr:
    """[A_0 | A_1 | ...]: same-height CSR tiles side by side, tile k's columns
    shifted by k * col_stride (the fused stationary-C operand, algos.hpp:378-415)."""
    if not tiles or len(tiles) > 16:
        raise ValueError("concat_cols: 1..16 tiles")
    t0 = tiles[0]
    if any(t.rows != t0.rows or t.dtype != t0.dtype for t in tiles):
        raise L.DimensionError("concat_cols: tiles differ in rows or dtype")
    nnz = sum(t.nnz for t in tiles)
    cols = col_stride * (len(tiles) - 1) + tiles[-1].cols
    out = DeviceCsr.empty(t0.rows, cols, nnz, dtype=t0.dtype, device=t0.device)
    K = len(tiles)
    rp = (C.c_void_p * K)(*[t.row_ptr.data_ptr() for t in tiles])
    ci = (C.c_void_p * K)(*[t.col_idx.data_ptr() if t.nnz else 0 for t in tiles])
    vv = (C.c_void_p * K)(*[t.values.data_ptr() if t.nnz else 0 for t in tiles])
    nz = (C.c_uint64 * K)(*[t.nnz for t in tiles])
    L.check(L.rdmm_csr_concat_cols(_wcode(t0.dtype), t0.rows, K, rp, ci, vv, nz, col_stride,
                                   out.row_ptr.data_ptr(), out.col_idx.data_ptr() if nnz else None,
                                   out.values.data_ptr() if nnz else None, _stream(stream)),
            "concat_cols")
    return out


def dense_add_into(c: torch.Tensor, x: torch.Tensor, stream=None) -> None:
    """c += x (tile.hpp:300-307)."""
    if c.shape != x.shape:
        raise L.DimensionError("dense_add_into: dimension mismatch")
    fn = L.rdmm_dense_add_into_f64 if c.dtype == torch.float64 else L.rdmm_dense_add_into_f32
    L.check(fn(c.shape[0], c.shape[1], c.data_ptr(), c.stride(0), x.data_ptr(), x.stride(0),
               _stream(stream)), "dense_add_into")


# ---------------------------------------------------------------- generators


def _finish(st, nnz, rows, cols, dtype, device) -> DeviceCsr:
    out = DeviceCsr.empty(rows, cols, nnz, dtype=dtype, device=device)
    L.check(L.rdmm_gen_finish(st, _wcode(dtype), out.row_ptr.data_ptr(),
                              out.col_idx.data_ptr() if nnz else None,
                              out.values.data_ptr() if nnz else None), "gen_finish")
    return out


def rmat(scale: int, edgefactor: int, seed: int = 1, a: float = 0.6, b: float = 0.4 / 3,
         c: float = 0.4 / 3, d: float = 0.4 / 3, multiplicity: bool = False,
         dtype=torch.float32, device="cuda") -> DeviceCsr:
    """R-MAT (gen.hpp:58-92) generated in device memory, bit-identical."""
    with torch.cuda.device(device):
        st = C.c_void_p()
        nnz = C.c_uint64(0)
        L.check(L.rdmm_gen_rmat_begin(a, b, c, d, scale, edgefactor, seed, int(multiplicity),
                                      C.byref(st), C.byref(nnz)), "rmat")
        n = 1 << scale
        return _finish(st, nnz.value, n, n, dtype, device)


def uniform_tiles(m: int, k: int, p: int, d: float, seed: int, dtype=torch.float32,
                  device="cuda") -> DeviceCsr:
    """uniform_tiles (gen.hpp:97-133) generated in device memory."""
    with torch.cuda.device(device):
        st = C.c_void_p()
        nnz = C.c_uint64(0)
        L.check(L.rdmm_gen_uniform_tiles_begin(m, k, p, d, seed, C.byref(st), C.byref(nnz)),
                "uniform_tiles")
        return _finish(st, nnz.value, m, k, dtype, device)


def permute_symmetric(a: DeviceCsr, seed: int, stream=None) -> DeviceCsr:
    """P A P^T with the reference's Fisher-Yates permutation (gen.hpp:134-155),
    relabelled and row-sorted on the device; bit-identical to the reference."""
    out = DeviceCsr.empty(a.rows, a.cols, a.nnz, dtype=a.dtype, device=a.device)
    L.check(L.rdmm_permute_symmetric(a.rows, a.cols, a.nnz, a.row_ptr.data_ptr(),
                                     a.col_idx.data_ptr(), a.values.data_ptr(), _wcode(a.dtype),
                                     seed, out.row_ptr.data_ptr(), out.col_idx.data_ptr(),
                                     out.values.data_ptr(), _stream(stream)),
            "permute_symmetric")
    return out


def permutation(n: int, seed: int):
    """The permutation alone (host): perm[old] = new (gen.hpp:141-147)."""
    import numpy as np

    perm = np.empty(n, np.uint32)
    L.check(L.rdmm_permutation(n, seed, perm.ctypes.data), "permutation")
    return perm


def random_dense(rows: int, cols: int, seed: int, max_value: int = 3, dtype=torch.float32,
                 device="cuda", stream=None) -> torch.Tensor:
    """random_dense (gen.hpp:174-181)."""
    out = torch.empty((rows, cols), dtype=dtype, device=device)
    L.check(L.rdmm_gen_random_dense(rows * cols, seed, max_value, _wcode(dtype),
                                    out.data_ptr(), _stream(stream)), "random_dense")
    return out


def real_twin(n: int, seed: int, dtype=torch.float32, device="cuda", stream=None):
    """Real-valued parity twin values 2*u01(seed, i) - 1."""
    out = torch.empty(n, dtype=dtype, device=device)
    L.check(L.rdmm_gen_real_twin(n, seed, _wcode(dtype), out.data_ptr(), _stream(stream)),
            "real_twin")
    return out


def rng_at(seed: int, first: int, count: int, device="cuda") -> torch.Tensor:
    out = torch.empty(count, dtype=torch.int64, device=device)
    L.check(L.rdmm_gen_rng_at(seed, first, count, out.data_ptr(),
                              _stream(None)), "rng_at")
    return out
