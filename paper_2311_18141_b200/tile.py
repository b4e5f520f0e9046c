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
               workspace: torch.Tensor | None = None) -> FlopMeter:
    """c += a @ b on the device; tile.hpp:170-188.  Raises DimensionError on
    mismatch exactly like the reference (tile.hpp:173-174)."""
    if a.cols != b.shape[0] or c.shape[0] != a.rows or c.shape[1] != b.shape[1]:
        raise L.DimensionError("spmm_local: dimension mismatch")
    if b.dtype != a.dtype or c.dtype != a.dtype:
        raise L.InvalidArgument("spmm_local: dtype mismatch")
    if b.stride(1) != 1 or c.stride(1) != 1:
        raise L.InvalidArgument("spmm_local: B and C must be row-major")
    n = b.shape[1]
    fl = C.c_uint64(0)
    fn = L.rdmm_spmm_csr_f64 if a.dtype == torch.float64 else L.rdmm_spmm_csr_f32
    ws = workspace.data_ptr() if workspace is not None else None
    wsb = workspace.numel() * workspace.element_size() if workspace is not None else 0
    L.check(fn(a.rows, a.cols, n, a.nnz, a.row_ptr.data_ptr(), a.col_idx.data_ptr(),
               a.values.data_ptr(), b.data_ptr(), b.stride(0), c.data_ptr(), c.stride(0),
               ws, wsb, _stream(stream), C.byref(fl)), "spmm_local")
    return FlopMeter(fl.value, c.shape[0] * c.shape[1])


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
