"""TEST INFRASTRUCTURE ONLY -- ctypes front-end for the CPU oracles.

Two implementations behind one interface:

* ``port()``  -- oracle/_build/librdmm_oracle.so, the plain-C restatement of
  the reference algorithms (oracle/rdmm_oracle.c).
* ``ref()``   -- oracle/_ref/librdmm_ref.so, the UNMODIFIED reference headers
  (/root/reference/proj/include/rdmm/*.hpp) compiled in place behind
  oracle/ref_shim.cpp.  Absent on a box where it was never built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this module; the product path (paper_2311_18141_b200) never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "librdmm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librdmm_ref.so")

VARIANTS = {
    "summa_bsp": 0,
    "stationary_c": 1,
    "stationary_a": 2,
    "stationary_b": 3,
    "ws_random": 4,
    "ws_locality": 5,
}


class OrcCsr(C.Structure):
    _fields_ = [
        ("rows", C.c_uint32),
        ("cols", C.c_uint32),
        ("nnz", C.c_uint64),
        ("dtype", C.c_int),
        ("row_ptr", C.POINTER(C.c_uint32)),
        ("col_idx", C.POINTER(C.c_uint32)),
        ("values", C.c_void_p),
    ]


class RefReport(C.Structure):
    _fields_ = [
        ("wall_seconds", C.c_double),
        ("max_total_seconds", C.c_double),
        ("checksum", C.c_double),
        ("total_flops", C.c_uint64),
        ("total_multiplies", C.c_uint64),
        ("total_steals", C.c_uint64),
        ("nranks", C.c_uint64),
        ("multiplies", C.c_uint64 * 64),
        ("flops", C.c_uint64 * 64),
        ("steals", C.c_uint64 * 64),
        ("steals_local", C.c_uint64 * 64),
        ("pushes", C.c_uint64 * 64),
        ("pops", C.c_uint64 * 64),
        ("total_seconds", C.c_double * 64),
    ]


@dataclass
class Csr:
    """Host CSR tile (reference CsrTile, tile.hpp:57-118)."""

    rows: int
    cols: int
    row_ptr: np.ndarray  # uint32, rows+1
    col_idx: np.ndarray  # uint32, nnz
    values: np.ndarray  # float32/float64, nnz

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    @property
    def dtype(self):
        return self.values.dtype

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.rows, self.cols), dtype=np.float64)
        r = np.repeat(np.arange(self.rows), np.diff(self.row_ptr.astype(np.int64)))
        np.add.at(d, (r, self.col_idx.astype(np.int64)), self.values.astype(np.float64))
        return d

    def rows_slice(self, r0: int, r1: int) -> "Csr":
        s, e = int(self.row_ptr[r0]), int(self.row_ptr[r1])
        return Csr(r1 - r0, self.cols, (self.row_ptr[r0:r1 + 1] - s).astype(np.uint32),
                   self.col_idx[s:e].copy(), self.values[s:e].copy())


def _wcode(dtype) -> int:
    return 8 if np.dtype(dtype) == np.float64 else 4


def _np_of(dt: int):
    return np.float64 if dt == 8 else np.float32


def as_orc(a: Csr) -> tuple[OrcCsr, tuple]:
    rp = np.ascontiguousarray(a.row_ptr, dtype=np.uint32)
    ci = np.ascontiguousarray(a.col_idx, dtype=np.uint32)
    vv = np.ascontiguousarray(a.values)
    o = OrcCsr(a.rows, a.cols, a.nnz, _wcode(vv.dtype),
               rp.ctypes.data_as(C.POINTER(C.c_uint32)),
               ci.ctypes.data_as(C.POINTER(C.c_uint32)), vv.ctypes.data)
    return o, (rp, ci, vv)  # keep-alive


class _Impl:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.p = prefix
        self.path = path
        L = self.lib
        P = C.POINTER
        if prefix == "orc":
            L.orc_csr_free.argtypes = [P(OrcCsr)]
            self._free = L.orc_csr_free
        else:
            L.ref_csr_free.argtypes = [P(OrcCsr)]
            self._free = L.ref_csr_free
        self._fn("splitmix64", C.c_uint64, [C.c_uint64])
        self._fn("rmat", C.c_int, [C.c_double] * 4 + [C.c_uint32, C.c_uint32, C.c_uint64,
                                                       C.c_int, C.c_int, P(OrcCsr)])
        self._fn("uniform_tiles", C.c_int, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_double,
                                            C.c_uint64, C.c_int, P(OrcCsr)])
        self._fn("random_csr", C.c_int, [C.c_uint32, C.c_uint32, C.c_double, C.c_uint64,
                                         C.c_int, C.c_int, P(OrcCsr)])
        self._fn("random_dense", None, [C.c_uint32, C.c_uint32, C.c_uint64, C.c_int, C.c_int,
                                        C.c_void_p])
        self._fn("permute_symmetric", C.c_int, [P(OrcCsr), C.c_uint64, P(OrcCsr)])
        self._fn("spgemm_flops", C.c_uint64, [P(OrcCsr), P(OrcCsr)])
        self._fn("csr_add", C.c_int, [P(OrcCsr), P(OrcCsr), P(OrcCsr)])
        if prefix == "orc":
            self._fn("spmm_rows", C.c_uint64, [P(OrcCsr), C.c_uint32, C.c_uint32, C.c_uint32,
                                               C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64])
            self._fn("spmm_local", C.c_uint64, [P(OrcCsr), C.c_uint32, C.c_uint32, C.c_void_p,
                                                C.c_uint64, C.c_void_p, C.c_uint64, P(C.c_int)])
            self._fn("spgemm_local", C.c_int, [P(OrcCsr), P(OrcCsr), C.c_uint32, C.c_uint32,
                                               P(OrcCsr), P(C.c_uint64)])
            self._fn("checksum_dense", C.c_double, [C.c_uint64, C.c_uint64, C.c_uint32,
                                                    C.c_uint32, C.c_void_p, C.c_int])
            self._fn("checksum_sparse", C.c_double, [P(OrcCsr), C.c_uint32, C.c_uint32])
            self._fn("csr_well_formed", C.c_int, [P(OrcCsr)])
            self._fn("dense_add_into", None, [C.c_uint64, C.c_void_p, C.c_void_p, C.c_int])
        else:
            self._fn("spmm_local", C.c_int, [P(OrcCsr), C.c_uint32, C.c_uint32, C.c_void_p,
                                             C.c_void_p, P(C.c_uint64)])
            self._fn("spgemm_local", C.c_int, [P(OrcCsr), P(OrcCsr), P(OrcCsr), P(C.c_uint64)])
            self._fn("hardware_concurrency", C.c_uint, [])
            self._fn("stage_imbalance", C.c_int, [P(OrcCsr), C.c_uint32, C.c_uint32]
                     + [P(C.c_double)] * 3 + [C.c_void_p])
            self._fn("read_matrix_market", C.c_int, [C.c_char_p, C.c_int, P(OrcCsr),
                                                     C.c_char_p, C.c_int])
            self._fn("roofline", C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_uint64,
                                           C.c_uint64, C.c_void_p])
            self._fn("imbalance_from_flops", None, [C.c_uint32, C.c_uint32, C.c_void_p,
                                                    P(C.c_double), P(C.c_double)])
            self._fn("run_multiply_spmm", C.c_int,
                     [C.c_int] * 5 + [C.c_uint64, C.c_double, C.c_double, C.c_uint32, C.c_uint32]
                     + [C.c_uint64] * 3 + [C.c_uint32] * 3
                     + [P(OrcCsr), C.c_void_p, C.c_void_p, C.c_uint64, P(RefReport)])
            self._fn("run_multiply_spgemm", C.c_int,
                     [C.c_int] * 5 + [C.c_uint64, C.c_double, C.c_double, C.c_uint32, C.c_uint32]
                     + [C.c_uint64] * 3 + [C.c_uint32] * 3
                     + [P(OrcCsr), P(OrcCsr), P(OrcCsr), P(OrcCsr), C.c_uint64, P(RefReport)])

    def _fn(self, name, res, args):
        f = getattr(self.lib, f"{self.p}_{name}")
        f.restype = res
        f.argtypes = args
        setattr(self, "_" + name, f)

    # -- helpers ---------------------------------------------------------
    def _take(self, o: OrcCsr) -> Csr:
        dt = _np_of(o.dtype)
        rp = np.ctypeslib.as_array(o.row_ptr, shape=(o.rows + 1,)).copy()
        n = int(o.nnz)
        ci = np.ctypeslib.as_array(o.col_idx, shape=(n,)).copy() if n else np.zeros(0, np.uint32)
        if n:
            buf = (C.c_char * (n * np.dtype(dt).itemsize)).from_address(o.values)
            vv = np.frombuffer(buf, dtype=dt).copy()
        else:
            vv = np.zeros(0, dt)
        self._free(C.byref(o))
        return Csr(int(o.rows), int(o.cols), rp.astype(np.uint32), ci.astype(np.uint32), vv)

    @staticmethod
    def _check(rc, what):
        if rc != 0:
            raise ValueError(f"{what} failed with code {rc}")

    # -- generators (gen.hpp) -------------------------------------------
    def splitmix64(self, x: int) -> int:
        return int(self._splitmix64(x))

    def rmat(self, scale, edgefactor, seed=1, a=0.6, b=0.4 / 3, c=0.4 / 3, d=0.4 / 3,
             multiplicity=False, dtype=np.float32) -> Csr:
        o = OrcCsr()
        self._check(self._rmat(a, b, c, d, scale, edgefactor, seed, int(multiplicity),
                               _wcode(dtype), C.byref(o)), "rmat")
        return self._take(o)

    def uniform_tiles(self, m, k, p, d, seed, dtype=np.float32) -> Csr:
        o = OrcCsr()
        self._check(self._uniform_tiles(m, k, p, d, seed, _wcode(dtype), C.byref(o)),
                    "uniform_tiles")
        return self._take(o)

    def random_csr(self, rows, cols, density, seed, max_value=3, dtype=np.float32) -> Csr:
        o = OrcCsr()
        self._check(self._random_csr(rows, cols, density, seed, max_value, _wcode(dtype),
                                     C.byref(o)), "random_csr")
        return self._take(o)

    def random_dense(self, rows, cols, seed, max_value=3, dtype=np.float32) -> np.ndarray:
        out = np.empty((rows, cols), dtype=dtype)
        self._random_dense(rows, cols, seed, max_value, _wcode(dtype), out.ctypes.data)
        return out

    def permute_symmetric(self, m: Csr, seed: int) -> Csr:
        a, keep = as_orc(m)
        o = OrcCsr()
        self._check(self._permute_symmetric(C.byref(a), seed, C.byref(o)), "permute")
        return self._take(o)

    # -- kernels (tile.hpp) ---------------------------------------------
    def spmm_local(self, a: Csr, b: np.ndarray, c: np.ndarray) -> int:
        """c += a @ b in place; returns flops (tile.hpp:170-188)."""
        assert b.flags.c_contiguous and c.flags.c_contiguous
        ao, keep = as_orc(a)
        n = b.shape[1]
        if self.p == "orc":
            err = C.c_int(0)
            f = self._spmm_local(C.byref(ao), b.shape[0], n, b.ctypes.data, n, c.ctypes.data,
                                 c.shape[1], C.byref(err))
            if err.value:
                raise ValueError("spmm_local: dimension mismatch")
            return int(f)
        fl = C.c_uint64(0)
        self._check(self._spmm_local(C.byref(ao), b.shape[0], n, b.ctypes.data, c.ctypes.data,
                                     C.byref(fl)), "spmm_local")
        return int(fl.value)

    def spmm_rows(self, a: Csr, r0: int, r1: int, b: np.ndarray, c: np.ndarray) -> int:
        ao, keep = as_orc(a)
        n = b.shape[1]
        return int(self._spmm_rows(C.byref(ao), r0, r1, n, b.ctypes.data, n, c.ctypes.data,
                                   c.shape[1]))

    def spgemm_local(self, a: Csr, b: Csr, r0: int = 0, r1: int | None = None):
        ao, k1 = as_orc(a)
        bo, k2 = as_orc(b)
        o = OrcCsr()
        fl = C.c_uint64(0)
        if self.p == "orc":
            rc = self._spgemm_local(C.byref(ao), C.byref(bo), r0,
                                    a.rows if r1 is None else r1, C.byref(o), C.byref(fl))
        else:
            assert r0 == 0 and r1 is None
            rc = self._spgemm_local(C.byref(ao), C.byref(bo), C.byref(o), C.byref(fl))
        self._check(rc, "spgemm_local")
        return self._take(o), int(fl.value)

    def spgemm_flops(self, a: Csr, b: Csr) -> int:
        ao, k1 = as_orc(a)
        bo, k2 = as_orc(b)
        return int(self._spgemm_flops(C.byref(ao), C.byref(bo)))

    def csr_add(self, a: Csr, b: Csr) -> Csr:
        ao, k1 = as_orc(a)
        bo, k2 = as_orc(b)
        o = OrcCsr()
        self._check(self._csr_add(C.byref(ao), C.byref(bo), C.byref(o)), "csr_add")
        return self._take(o)

    def stage_imbalance(self, a: Csr, grid: int, stages: int = 0) -> dict:
        ao, keep = as_orc(a)
        K = stages or grid
        fl = np.zeros((grid * grid, K), np.uint64)
        ps, e2e, nb = C.c_double(), C.c_double(), C.c_double()
        self._check(self._stage_imbalance(C.byref(ao), grid, stages, C.byref(ps), C.byref(e2e),
                                          C.byref(nb), fl.ctypes.data), "stage_imbalance")
        return {"per_stage_flop_imbalance": ps.value, "end_to_end_flop_imbalance": e2e.value,
                "nnz_imbalance": nb.value, "stage_flops": fl.astype(np.int64)}

    def imbalance_from_flops(self, f: np.ndarray) -> dict:
        f = np.ascontiguousarray(f, np.uint64)
        ps, e2e = C.c_double(), C.c_double()
        self._imbalance_from_flops(f.shape[0], f.shape[1], f.ctypes.data, C.byref(ps),
                                   C.byref(e2e))
        return {"per_stage_flop_imbalance": ps.value, "end_to_end_flop_imbalance": e2e.value}

    def read_matrix_market(self, path: str, dtype=np.float32):
        """-> Csr, or raises ValueError(message) on the reference's mmio_error."""
        o = OrcCsr()
        msg = C.create_string_buffer(512)
        rc = self._read_matrix_market(str(path).encode(), np.dtype(dtype).itemsize, C.byref(o),
                                      msg, 512)
        if rc == 8:
            raise ValueError(msg.value.decode())
        self._check(rc, "read_matrix_market")
        return self._take(o)

    def roofline(self, shape, cost, spgemm=False, flops=0, out_nnz=0) -> np.ndarray:
        sh = np.asarray(shape, np.float64)
        co = np.asarray(cost, np.float64)
        out = np.zeros(7)
        self._check(self._roofline(sh.ctypes.data, co.ctypes.data, int(spgemm), flops, out_nnz,
                                   out.ctypes.data), "roofline")
        return out

    def checksum_dense(self, g: np.ndarray, tm: int, tn: int) -> float:
        return float(self._checksum_dense(g.shape[0], g.shape[1], tm, tn, g.ctypes.data,
                                          _wcode(g.dtype)))

    def checksum_sparse(self, g: Csr, tm: int, tn: int) -> float:
        go, keep = as_orc(g)
        return float(self._checksum_sparse(C.byref(go), tm, tn))

    def well_formed(self, g: Csr) -> bool:
        go, keep = as_orc(g)
        return bool(self._csr_well_formed(C.byref(go)))

    # -- reference driver (algos.hpp:673-752) ----------------------------
    def run_multiply_spmm(self, a: Csr, b: np.ndarray, c: np.ndarray, *, variant="stationary_c",
                          ws_base="stationary_a", prefetch=True, offset=True, seed=0,
                          delay_ns_per_flop=0.0, random_delay_ms=0.0, grid=(1, 1), tiles=None,
                          heap_bytes=0) -> RefReport:
        m, k = a.rows, a.cols
        n = b.shape[1]
        tm, tk, tn = tiles or (-(-m // grid[0]), -(-k // grid[1]), -(-n // grid[1]))
        ao, keep = as_orc(a)
        rep = RefReport()
        rc = self._run_multiply_spmm(_wcode(b.dtype), VARIANTS[variant], VARIANTS[ws_base],
                                     int(prefetch), int(offset), seed, delay_ns_per_flop,
                                     random_delay_ms, grid[0], grid[1], m, k, n, tm, tk, tn,
                                     C.byref(ao), b.ctypes.data, c.ctypes.data, heap_bytes,
                                     C.byref(rep))
        self._check(rc, "run_multiply_spmm")
        return rep

    def run_multiply_spgemm(self, a: Csr, b: Csr, c0: Csr, *, variant="stationary_c",
                            ws_base="stationary_a", prefetch=True, offset=True, seed=0,
                            delay_ns_per_flop=0.0, random_delay_ms=0.0, grid=(1, 1), tiles=None,
                            heap_bytes=0):
        m, k, n = a.rows, a.cols, b.cols
        tm, tk, tn = tiles or (-(-m // grid[0]), -(-k // grid[1]), -(-n // grid[1]))
        ao, k1 = as_orc(a)
        bo, k2 = as_orc(b)
        co, k3 = as_orc(c0)
        o = OrcCsr()
        rep = RefReport()
        rc = self._run_multiply_spgemm(_wcode(a.values.dtype), VARIANTS[variant],
                                       VARIANTS[ws_base], int(prefetch), int(offset), seed,
                                       delay_ns_per_flop, random_delay_ms, grid[0], grid[1],
                                       m, k, n, tm, tk, tn, C.byref(ao), C.byref(bo),
                                       C.byref(co), C.byref(o), heap_bytes, C.byref(rep))
        self._check(rc, "run_multiply_spgemm")
        return self._take(o), rep


_port = None
_ref = None


def build() -> None:
    """Compile the oracle (and the reference shim where the headers exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def port() -> _Impl:
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        _port = _Impl(PORT_SO, "orc")
    return _port


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> _Impl:
    global _ref
    if _ref is None:
        _ref = _Impl(REF_SO, "ref")
    return _ref


# -- vectorised counter RNG (gen.hpp:20-34), for real-valued parity twins ---
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64_np(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
    x = (x ^ (x >> np.uint64(30))) * _M1
    x = (x ^ (x >> np.uint64(27))) * _M2
    return x ^ (x >> np.uint64(31))


def rng_at_np(seed: int, counters: np.ndarray) -> np.ndarray:
    base = np.array([seed], dtype=np.uint64) * np.uint64(0x2545F4914F6CDD1D)
    return splitmix64_np(base + counters.astype(np.uint64))


def u01_np(seed: int, counters: np.ndarray) -> np.ndarray:
    return (rng_at_np(seed, counters) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53


def real_twin(n: int, seed: int, dtype=np.float32) -> np.ndarray:
    """SURVEY §8(d) real-valued twin: 2*u01(seed, idx) - 1 (U(-1,1))."""
    return (2.0 * u01_np(seed, np.arange(n, dtype=np.uint64)) - 1.0).astype(dtype)
