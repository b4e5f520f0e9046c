"""World-size-2 multi-process checks of the fabric's control plane on CPU
(gloo for the rendezvous): two processes share one control segment by
session name, as the torchrun bench does with one process per GPU.  The
ranks are control-plane-only (device -1, no heap), so no GPU is needed.

Mirrors test_fabric.cpp:188-210 (fetch_add linearisability), :250-278
(queue exactly-once), :280-295 (barrier)."""
import ctypes as C
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2311_18141_b200._lib as L

    name = [f"t{os.getpid()}_{port}" if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    dev = (C.c_int * 1)(-1)
    cfg = L.FabricConfig(world, 6, 0, 1024, 8 << 20, rank, 1, dev, name[0].encode())
    f = C.c_void_p()
    L.check(L.rdmm_fabric_create(C.byref(cfg), C.byref(f)), "create")
    res = {}
    # fetch-add linearisability
    cell = L.Gptr()
    L.check(L.rdmm_ctrl_cells(f, rank, 77, 1, C.byref(cell)), "cells")
    L.check(L.rdmm_barrier(f, rank), "barrier")
    olds = []
    for _ in range(500):
        v = C.c_int64()
        L.check(L.rdmm_fetch_add_i64(f, rank, cell, 1, C.byref(v)), "fetch_add")
        olds.append(v.value)
    L.check(L.rdmm_barrier(f, rank), "barrier")
    allolds = [None] * world
    dist.all_gather_object(allolds, olds)
    res["olds"] = sorted(x for o in allolds for x in o)
    # queues: every rank pushes 64 entries into rank 0's queue
    q = (C.c_uint64 * world)()
    L.check(L.rdmm_queue_open(f, rank, 99, 256, q), "queue_open")
    L.check(L.rdmm_barrier(f, rank), "barrier")
    for n in range(64):
        g = L.Gptr(rank, 0, n, 0)
        payload = C.c_uint64(rank * 1000 + n)
        L.check(L.rdmm_queue_push(f, rank, q[0], g, C.byref(payload), 8), "push")
    L.check(L.rdmm_barrier(f, rank), "barrier")
    got = []
    if rank == 0:
        while True:
            g, inl, ok = L.Gptr(), C.c_uint64(), C.c_int()
            L.check(L.rdmm_queue_pop(f, rank, q[0], C.byref(g), C.byref(inl), 8, C.byref(ok)),
                    "pop")
            if not ok.value:
                break
            got.append((g.rank, g.offset, inl.value))
    else:
        g, inl, ok = L.Gptr(), C.c_uint64(), C.c_int()
        rc = L.rdmm_queue_pop(f, rank, q[0], C.byref(g), C.byref(inl), 8, C.byref(ok))
        res["non_owner_pop_rc"] = rc
    res["popped"] = got
    for _ in range(20):
        L.check(L.rdmm_barrier(f, rank), "barrier")
    L.rdmm_ctrl_release(f, rank, 77)
    L.rdmm_ctrl_release(f, rank, 99)
    L.rdmm_fabric_destroy(f)
    out[rank] = res
    dist.destroy_process_group()


def test_two_process_control_plane():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, port, out), nprocs=world, join=True,
                       start_method="spawn")
    assert out[0]["olds"] == list(range(1000))
    popped = out[0]["popped"]
    assert sorted(popped) == sorted((r, n, r * 1000 + n) for r in range(world) for n in range(64))
    assert out[1]["non_owner_pop_rc"] == 2  # RDMM_ERR_FABRIC: not the queue owner


def test_bench_session_and_layout():
    import bench

    class A:
        grid = None
        mtiles = ktiles = ntiles = 0

    # SpMM: 1 x P column split (every rank all rows, N/P columns, K = P)
    (pr, pc), tiles = bench.layout(bench.CONFIGS["cfg3"], 8, A)
    assert (pr, pc) == (1, 8) and tuple(tiles) == (4194304, 524288, 16)
    (pr, pc), tiles = bench.layout(bench.CONFIGS["cfg5"], 4, A)
    assert (pr, pc) == (1, 4) and tuple(tiles) == (4194304, 1048576, 64)
    (pr, pc), tiles = bench.layout(bench.CONFIGS["cfg3"], 1, A)
    assert (pr, pc) == (1, 1) and tuple(tiles) == (4194304, 4194304, 128)
    (pr, pc), tiles = bench.layout(bench.CONFIGS["cfg4"], 4, A)
    assert (pr, pc) == (2, 2) and tuple(tiles) == ((1 << 20) // 8, (1 << 20) // 2, (1 << 20) // 2)
    # cfg2: stationary variants on a square-ish grid (2x2 at 4, 4x2 at 8, 2x1 at 2)
    for P, grid in ((1, (1, 1)), (2, (2, 1)), (4, (2, 2)), (8, (4, 2))):
        (pr, pc), tiles = bench.layout(bench.CONFIGS["cfg2"], P, A)
        assert (pr, pc) == grid
        assert tuple(tiles) == ((1 << 17) // (4 * pr), (1 << 17) // pr, (1 << 17) // pc)
    assert bench.make_session(1, 0) is None


def test_bench_owned_tile_bytes():
    import bench

    class G:
        def __init__(self, pr, pc):
            self.pr, self.pc = pr, pc

        def owner(self, i, j):  # ProcGrid rule, distmat.hpp:20-36
            return (i % self.pr) * self.pc + (j % self.pc)

    # 10 x 6 fp32 in 4 x 4 tiles on a 2 x 1 grid: rank 0 owns tile rows 0 and 2
    assert bench.owned_dense_bytes(G(2, 1), 10, 6, 4, 4, 0) == (4 + 2) * 6 * 4
    assert bench.owned_dense_bytes(G(2, 1), 10, 6, 4, 4, 1) == 4 * 6 * 4
    # every element is owned exactly once
    g = G(2, 2)
    assert sum(bench.owned_dense_bytes(g, 10, 6, 4, 4, r) for r in range(4)) == 10 * 6 * 4
