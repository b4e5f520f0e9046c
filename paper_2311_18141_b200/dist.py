"""Python mirror of the reference's distributed API (Fabric, DistSparse,
DistDense, run_multiply -- /root/reference/proj/include/rdmm/{fabric,
distmat,algos}.hpp) over the host C-ABI in include/rdmm_host.h.

Every collective call drives all ranks hosted by this process (one thread
per local rank inside the library).  For one process per GPU (torchrun),
create the Fabric with first_local=rank, nlocal=1 and a shared `session`.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L

VARIANTS = ["summa_bsp", "stationary_c", "stationary_a", "stationary_b", "ws_random",
            "ws_locality"]
MAXR = 64


class Options(C.Structure):
    _fields_ = [("variant", C.c_int), ("ws_base", C.c_int), ("prefetch", C.c_int),
                ("offset", C.c_int), ("seed", C.c_uint64), ("delay_ns_per_flop", C.c_double),
                ("random_delay_ms_max", C.c_double), ("record_events", C.c_int),
                ("record_triples", C.c_int), ("lookahead", C.c_int),
                ("ws_local_inplace", C.c_int), ("checksum", C.c_int), ("fuse_k", C.c_int),
                ("split_local", C.c_int), ("time_stages", C.c_int), ("pipeline", C.c_int),
                ("row_blocks", C.c_int), ("deterministic", C.c_int)]


class Report(C.Structure):
    _fields_ = [("wall_seconds", C.c_double), ("checksum", C.c_double),
                ("total_flops", C.c_uint64), ("total_multiplies", C.c_uint64),
                ("total_steals", C.c_uint64), ("nranks", C.c_uint32)] + [
        (n, C.c_uint64 * MAXR) for n in ("multiplies", "flops", "output_nnz", "steals",
                                         "steals_local", "pushes", "pops", "bytes_self",
                                         "bytes_on_node", "bytes_off_node")] + [
        ("total_seconds", C.c_double * MAXR), ("ntriples", C.c_uint64),
        ("triples", C.POINTER(C.c_uint32)), ("nstages", C.c_uint32),
        ("stage_flops", C.POINTER(C.c_uint64)), ("stage_ms", C.POINTER(C.c_double))]


_u32, _u64, _vp, _int = C.c_uint32, C.c_uint64, C.c_void_p, C.c_int
_h = L.lib
_h.rdmm_h_fabric_create.argtypes = [_u32, _u64, _u32, _u64, _u32, _u32, C.POINTER(_int),
                                    C.c_char_p, C.POINTER(_vp)]
_h.rdmm_h_fabric_destroy.argtypes = [_vp]
_h.rdmm_h_fabric_destroy.restype = None
_h.rdmm_h_fabric_handle.argtypes = [_vp]
_h.rdmm_h_fabric_handle.restype = _vp
_h.rdmm_h_matrix_create.argtypes = [_vp, _int, _int, _u64, _u64, _u32, _u32, _u32, _u32, _int,
                                    C.POINTER(_vp)]
_h.rdmm_h_matrix_destroy.argtypes = [_vp]
_h.rdmm_h_matrix_destroy.restype = None
_h.rdmm_h_sparse_init.argtypes = [_vp, _vp, _vp, _vp, _u64, _int]
_h.rdmm_h_dense_init.argtypes = [_vp, _vp, _u64]
_h.rdmm_h_dense_to_host.argtypes = [_vp, _vp]
_h.rdmm_h_sparse_nnz.argtypes = [_vp, C.POINTER(_u64)]
_h.rdmm_h_sparse_to_host.argtypes = [_vp, _vp, _vp, _vp]
_h.rdmm_h_run_multiply.argtypes = [_vp, _vp, _vp, _vp, C.POINTER(Options), C.POINTER(Report)]
_h.rdmm_h_dense_zero.argtypes = [_vp]
_h.rdmm_h_dense_zero.restype = _int
_h.rdmm_h_dense_owned_to_host.argtypes = [_vp, _vp, _u64]
_h.rdmm_h_dense_owned_to_host.restype = _int
_h.rdmm_h_dense_owned_to_host_async.argtypes = [_vp, _vp, _u64, _vp]
_h.rdmm_h_dense_owned_to_host_async.restype = _int
_h.rdmm_h_sparse_owned_to_host.argtypes = [_vp, _vp, _u64, C.POINTER(_u64)]
_h.rdmm_h_sparse_owned_to_host.restype = _int
_h.rdmm_h_fabric_stream.argtypes = [_vp, _u32]
_h.rdmm_h_fabric_stream.restype = _vp
_h.rdmm_h_free.argtypes = [_vp]
_h.rdmm_h_free.restype = None
_h.rdmm_tile_fetches.argtypes = [_vp, _vp, _u64]
_h.rdmm_tile_fetches.restype = _u64
_h.rdmm_traffic_clear.argtypes = [_vp]
_h.rdmm_traffic_clear.restype = None
for _n in ("rdmm_h_fabric_create", "rdmm_h_matrix_create", "rdmm_h_sparse_init",
           "rdmm_h_dense_init", "rdmm_h_dense_to_host", "rdmm_h_sparse_nnz",
           "rdmm_h_sparse_to_host", "rdmm_h_run_multiply"):
    getattr(_h, _n).restype = _int


class TrafficRec(C.Structure):  # rdmm_traffic (fabric.hpp:89-203 TrafficLog cell)
    _fields_ = [("bytes_put", C.c_uint64), ("bytes_got", C.c_uint64), ("puts", C.c_uint64),
                ("gets", C.c_uint64), ("atomic_ops", C.c_uint64)]


_h.rdmm_traffic_pair.argtypes = [_vp, _u32, _u32, C.POINTER(TrafficRec)]
_h.rdmm_traffic_pair.restype = _int


class TileFetchRec(C.Structure):
    _fields_ = [("src", C.c_uint32), ("dst", C.c_uint32), ("label", C.c_int64),
                ("matrix", C.c_int32), ("i", C.c_uint32), ("j", C.c_uint32)]


@dataclass
class ProcGrid:
    """distmat.hpp:20-36"""

    pr: int = 1
    pc: int = 1

    def nranks(self):
        return self.pr * self.pc

    def owner(self, i, j):
        return (i % self.pr) * self.pc + (j % self.pc)


class Fabric:
    """fabric.hpp:205-412 (+ B200 placement: devices, first_local/nlocal,
    session)."""

    def __init__(self, nranks=1, heap_bytes=64 << 20, node_group=6, queue_capacity=4096,
                 devices=None, first_local=0, nlocal=0, session=None):
        self.nranks = nranks
        n = nlocal or nranks - first_local
        dev = (C.c_int * n)(*devices) if devices is not None else None
        h = C.c_void_p()
        L.check(_h.rdmm_h_fabric_create(nranks, heap_bytes, node_group, queue_capacity,
                                        first_local, nlocal, dev,
                                        session.encode() if session else None, C.byref(h)),
                "Fabric")
        self._h = h
        self._mats = []

    @property
    def handle(self):
        return _h.rdmm_h_fabric_handle(self._h)

    def stream(self, rank):
        """cudaStream_t (int) of a local rank's compute stream."""
        return _h.rdmm_h_fabric_stream(self._h, rank)

    def tile_fetches(self):
        n = _h.rdmm_tile_fetches(self.handle, None, 0)
        arr = (TileFetchRec * max(1, n))()
        _h.rdmm_tile_fetches(self.handle, arr, n)
        return [(r.src, r.dst, r.label, r.matrix, r.i, r.j) for r in arr[:n]]

    def traffic(self, src, dst):
        """Bytes and operations moved from rank `src` to rank `dst` as logged
        by this process (gets issued by dst, puts issued by src): the byte-exact
        TrafficLog of fabric.hpp:89-203."""
        t = TrafficRec()
        L.check(_h.rdmm_traffic_pair(self.handle, src, dst, C.byref(t)), "traffic")
        return dict(bytes_put=t.bytes_put, bytes_got=t.bytes_got, puts=t.puts, gets=t.gets,
                    atomic_ops=t.atomic_ops)

    def remote_bytes_in(self, rank):
        """Bytes `rank` received from other ranks (NVLink traffic into its GPU):
        its gets from peers plus peers' puts into it, as logged here."""
        tot = 0
        for r in range(self.nranks):
            if r == rank:
                continue
            t = self.traffic(r, rank)
            tot += t["bytes_got"] + t["bytes_put"]
        return tot

    def clear_traffic(self):
        _h.rdmm_traffic_clear(self.handle)

    def close(self):
        for m in self._mats:
            m.close()
        self._mats = []
        if self._h:
            _h.rdmm_h_fabric_destroy(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Mat:
    kind = 0

    def __init__(self, f: Fabric, m, n, tm, tn, grid: ProcGrid, matrix_id=0, dtype=np.float32):
        self.f, self.m, self.n, self.tm, self.tn, self.grid = f, m, n, tm, tn, grid
        self.dtype = np.dtype(dtype)
        h = C.c_void_p()
        L.check(_h.rdmm_h_matrix_create(f._h, self.kind, self.dtype.itemsize, m, n, tm, tn,
                                        grid.pr, grid.pc, matrix_id, C.byref(h)), "matrix")
        self._h = h
        f._mats.append(self)

    def close(self):
        if self._h:
            _h.rdmm_h_matrix_destroy(self._h)
            self._h = None

    @property
    def M(self):
        return -(-self.m // self.tm)

    @property
    def N(self):
        return -(-self.n // self.tn)


class DistSparse(_Mat):
    """distmat.hpp:210-398"""

    kind = 0

    def init(self):
        L.check(_h.rdmm_h_sparse_init(self._h, None, None, None, 0, 0), "init")

    def init_from_global(self, row_ptr, col_idx, values):
        rp = np.ascontiguousarray(row_ptr, dtype=np.uint32)
        ci = np.ascontiguousarray(col_idx, dtype=np.uint32)
        vv = np.ascontiguousarray(values, dtype=self.dtype)
        L.check(_h.rdmm_h_sparse_init(self._h, rp.ctypes.data, ci.ctypes.data, vv.ctypes.data,
                                      len(ci), 0), "init_from_global")

    def init_from_device(self, dcsr):
        """B200: tiles cut on the device from a DeviceCsr (any local GPU)."""
        L.check(_h.rdmm_h_sparse_init(self._h, dcsr.row_ptr.data_ptr(),
                                      dcsr.col_idx.data_ptr() if dcsr.nnz else None,
                                      dcsr.values.data_ptr() if dcsr.nnz else None, dcsr.nnz, 1),
                "init_from_device")

    def owned_bytes(self):
        n = C.c_uint64(0)
        L.check(_h.rdmm_h_sparse_owned_to_host(self._h, None, 0, C.byref(n)), "owned_bytes")
        return n.value

    def owned_to_host(self, buf):
        """D2H of this process's tiles (raw CSR arrays) into `buf` (a pinned
        uint8 tensor or numpy array); returns bytes moved."""
        ptr = buf.data_ptr() if hasattr(buf, "data_ptr") else buf.ctypes.data
        cap = buf.numel() if hasattr(buf, "numel") else buf.nbytes
        n = C.c_uint64(0)
        L.check(_h.rdmm_h_sparse_owned_to_host(self._h, ptr, cap, C.byref(n)), "owned_to_host")
        return n.value

    def nnz(self):
        n = C.c_uint64(0)
        L.check(_h.rdmm_h_sparse_nnz(self._h, C.byref(n)), "nnz")
        return n.value

    def to_global(self):
        nnz = self.nnz()
        rp = np.zeros(self.m + 1, np.uint32)
        ci = np.zeros(max(nnz, 1), np.uint32)
        vv = np.zeros(max(nnz, 1), self.dtype)
        L.check(_h.rdmm_h_sparse_to_host(self._h, rp.ctypes.data, ci.ctypes.data,
                                         vv.ctypes.data), "to_global")
        return rp, ci[:nnz], vv[:nnz]


class DistDense(_Mat):
    """distmat.hpp:92-205"""

    kind = 1

    def init(self):
        L.check(_h.rdmm_h_dense_init(self._h, None, 0), "init")

    def init_from_global(self, global_array):
        g = np.ascontiguousarray(global_array, dtype=self.dtype)
        assert g.shape == (self.m, self.n)
        L.check(_h.rdmm_h_dense_init(self._h, g.ctypes.data, self.n), "init_from_global")

    def init_from_device(self, tensor):
        """B200: scatter from a device (or pinned host) tensor, row-major;
        re-initialisation reuses the tiles in place."""
        assert tuple(tensor.shape) == (self.m, self.n) and tensor.stride(1) == 1
        L.check(_h.rdmm_h_dense_init(self._h, tensor.data_ptr(), tensor.stride(0)),
                "init_from_device")

    def zero(self):
        L.check(_h.rdmm_h_dense_zero(self._h), "zero")

    def owned_to_host(self, out):
        """D2H of this process's tiles into `out` (m x n row-major, e.g. a
        pinned tensor or numpy array); returns bytes moved."""
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        L.check(_h.rdmm_h_dense_owned_to_host(self._h, ptr, self.n), "owned_to_host")

    def owned_to_host_async(self, out, stream):
        """Enqueue the D2H of this process's tiles into `out` on `stream` (a
        torch.cuda.Stream or raw cudaStream_t on the rank's device) after the
        rank's queued compute, without waiting."""
        ptr = out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data
        sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        L.check(_h.rdmm_h_dense_owned_to_host_async(self._h, ptr, self.n, sp),
                "owned_to_host_async")

    def to_global(self):
        out = np.zeros((self.m, self.n), self.dtype)
        L.check(_h.rdmm_h_dense_to_host(self._h, out.ctypes.data), "to_global")
        return out


@dataclass
class RunReport:
    """algos.hpp:73-96 (per-rank arrays cover this process's ranks)."""

    wall_seconds: float
    checksum: float
    total_flops: int
    total_multiplies: int
    total_steals: int
    per_rank: list = field(default_factory=list)
    triples: list = field(default_factory=list)
    # flops per rank per k tile step (RankStats::stage_flops), int64 [P, K]
    stage_flops: np.ndarray = field(default_factory=lambda: np.zeros((0, 0), np.int64))
    # device ms per rank per k tile step (RankStats::stage_ms, time_stages=True)
    stage_ms: np.ndarray | None = None

    def imbalance(self):
        """Per-stage and end-to-end flop imbalance of this run
        (analytics.hpp:66-90 over the multiply's own flop table)."""
        from .analytics import imbalance_from_flops
        return imbalance_from_flops(self.stage_flops)


def run_multiply(f: Fabric, A: DistSparse, B, Cm, variant="stationary_c", ws_base="stationary_a",
                 prefetch=True, offset=True, seed=0, delay_ns_per_flop=0.0,
                 random_delay_ms_max=0.0, record_events=True, record_triples=False,
                 lookahead=2, ws_local_inplace=True, checksum=True, fuse_k=True,
                 split_local=True, time_stages=False, pipeline=True, row_blocks=0,
                 deterministic=False) -> RunReport:
    """C += A*B on the fabric -- algos.hpp:673-752."""
    o = Options(VARIANTS.index(variant), VARIANTS.index(ws_base), int(prefetch), int(offset),
                seed, delay_ns_per_flop, random_delay_ms_max, int(record_events),
                int(record_triples), lookahead, int(ws_local_inplace), int(checksum),
                int(fuse_k), int(split_local), int(time_stages), int(pipeline), int(row_blocks),
                int(deterministic))
    r = Report()
    L.check(_h.rdmm_h_run_multiply(f._h, A._h, B._h, Cm._h, C.byref(o), C.byref(r)),
            "run_multiply")
    per = []
    for p in range(r.nranks):
        per.append(dict(multiplies=r.multiplies[p], flops=r.flops[p], output_nnz=r.output_nnz[p],
                        steals=r.steals[p], steals_with_local_component=r.steals_local[p],
                        queue_pushes=r.pushes[p], queue_pops=r.pops[p],
                        bytes_self=r.bytes_self[p], bytes_on_node=r.bytes_on_node[p],
                        bytes_off_node=r.bytes_off_node[p], total_seconds=r.total_seconds[p]))
    tr = []
    if r.ntriples:
        a = np.ctypeslib.as_array(r.triples, shape=(r.ntriples * 4,)).reshape(-1, 4).copy()
        tr = [tuple(int(x) for x in row) for row in a]
        _h.rdmm_h_free(r.triples)
    sf = np.zeros((r.nranks, r.nstages), np.int64)
    if r.nstages and r.stage_flops:
        sf[:] = np.ctypeslib.as_array(r.stage_flops, shape=(r.nranks * r.nstages,)).reshape(
            r.nranks, r.nstages)
        _h.rdmm_h_free(r.stage_flops)
    sm = None
    if r.nstages and r.stage_ms:
        sm = np.ctypeslib.as_array(r.stage_ms, shape=(r.nranks * r.nstages,)).reshape(
            r.nranks, r.nstages).copy()
        _h.rdmm_h_free(r.stage_ms)
    return RunReport(r.wall_seconds, r.checksum, r.total_flops, r.total_multiplies,
                     r.total_steals, per, tr, sf, sm)
